// Host-side runtime of the B200 CVO engine: device contexts, uploaded clouds,
// pair-list workspaces and the batched "round" executor that the solver
// drives (one round = batched builds + batched sweeps + one D2H).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <atomic>
#include <cstdint>
#include <exception>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <utility>
#include <string>
#include <vector>

#include "../../include/kreg_b200.h"
#include "engine.cuh"

namespace kreg_host {

// NVTX range for the duration of a scope (SURVEY.md §5 tracing): rounds,
// their launch / wait phases and whole solver calls show up on the host
// timeline of nsys / ncu --nvtx (a no-op without an attached tool).
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};

// Exception carrying a kreg_status; the C-ABI maps it back to a code.
struct Error : std::runtime_error {
  kreg_status code;
  Error(kreg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what);
#define KREG_CUDA(call)                                   \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) ::kreg_host::throw_cuda(e_, #call); \
  } while (0)

// device allocation accounting (count, bytes) — cudaMalloc/cudaFree synchronise
inline long long g_device_allocs = 0;
inline long long g_device_alloc_bytes = 0;
inline double g_device_alloc_seconds = 0.0;  // host time spent in cudaFree/cudaMalloc/cudaMemset of DevBuf

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr && owned) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    owned = true;
  }
  bool owned = true;  // false: points into memory owned elsewhere (a context arena)
  void swap(DevBuf& o) {
    std::swap(ptr, o.ptr);
    std::swap(cap, o.cap);
    std::swap(owned, o.owned);
  }
  void borrow(T* p, size_t n) {
    release();
    ptr = p;
    cap = n;
    owned = false;
  }
  // grow (discarding contents) to hold at least n elements; optional zero fill
  void ensure(size_t n, bool zero = false, double slack = 1.25) {
    if (n <= cap && ptr) return;
    const auto t0 = std::chrono::steady_clock::now();
    release();
    size_t want = n < 16 ? 16 : static_cast<size_t>(static_cast<double>(n) * slack);
    ++g_device_allocs;
    g_device_alloc_bytes += static_cast<long long>(want * sizeof(T));
    static const bool trace = std::getenv("KREG_TRACE_ALLOC") != nullptr;
    if (trace) std::fprintf(stderr, "kreg-alloc elem=%zu n=%zu old_cap=%zu\n", sizeof(T), want, cap);
    cudaError_t e = cudaMalloc(&ptr, want * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      ptr = nullptr;
      throw Error(KREG_OUT_OF_MEMORY, "device allocation of " + std::to_string(want * sizeof(T)) + " bytes failed");
    }
    cap = want;
    if (zero) KREG_CUDA(cudaMemset(ptr, 0, want * sizeof(T)));
    g_device_alloc_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};

template <typename T>
struct PinnedBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  ~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
  }
  void ensure(size_t n) {
    if (n <= cap && ptr) return;
    if (ptr) cudaFreeHost(ptr);
    size_t want = n < 16 ? 16 : n + n / 4;
    KREG_CUDA(cudaMallocHost(&ptr, want * sizeof(T)));
    cap = want;
  }
};

struct ChannelInfo {
  std::string name;
  int dim;
  int kind;
};

struct Params {  // flattened KernelParams (kernels.hpp:23-33)
  double sigma = 1.0;
  double lengthscale = 1.0;
  std::vector<kreg_channel_params> per_channel;
};

struct Config {  // RegistrationConfig (registration.hpp:13-40)
  kreg_registration_config c;
};

struct RoundSlot;

// Cross-rank combination of one round's results (row sharding, solver.cpp).
struct Collective {
  kreg_collective_fn fn = nullptr;
  void* user = nullptr;
};

// Native NCCL collective (nccl_coll.cpp): installed as a context's collective.
struct NcclState;
void nccl_unique_id(unsigned char out[128]);
void nccl_attach(kreg_ctx* ctx, const unsigned char id[128], int rank, int world, bool deterministic);
void nccl_detach(kreg_ctx* ctx);
void nccl_free(NcclState* s);
long long nccl_calls(const kreg_ctx* ctx);

}  // namespace kreg_host

struct kreg_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  bool profiling = false;
  double sweep_ms = 0.0;
  long long sweep_launches = 0;
  long long sweep_issued = 0;  // sweep launches issued, re-runs included
  long long pair_evals = 0;
  long long pairs_streamed = 0;
  long long slots_streamed = 0;
  long long launches_base = 0;
  // round staging: slots 0 and 1 alternate in the batched solver (one round
  // in flight on the device while the host plans the other), slot 2 serves
  // the synchronous calls
  // (slots 3-5: groups 0, 2, 3 of a multi-group batch, on their own streams like slot 1)
  kreg_host::RoundSlot* rs[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  kreg_host::DevBuf<double> d_T2;
  kreg_host::DevBuf<unsigned long long> d_disp;
  // end-to-end calls: pinned host staging and device arena of their clouds
  kreg_host::PinnedBuf<double> stage_d;
  kreg_host::PinnedBuf<float> stage_f;
  kreg_host::DevBuf<double> arena_d;
  kreg_host::DevBuf<float> arena_f;
  kreg_host::DevBuf<double4> arena_w;
  // frame ingest (kreg_depth_rgb_to_cloud / kreg_select_points)
  kreg_host::DevBuf<uint8_t> ing_rgb, ing_valid_in, ing_score, ing_valid;
  kreg_host::DevBuf<uint16_t> ing_depth;
  kreg_host::DevBuf<float> ing_sem;
  kreg_host::DevBuf<unsigned long long> ing_hist;
  kreg_host::DevBuf<int> ing_block_count, ing_pixels;
  kreg_host::DevBuf<long long> ing_block_off;
  kreg_host::DevBuf<double> ing_xyz, ing_feat;
  // pair-list workspaces kept across registrations (device buffers keep capacity)
  std::vector<kreg_pairs*> pool;
  int max_active = 0;  // lockstep window of kreg_register_batch (0 = all at once)
  // candidate-list radius R_s = cutoff (1 + skin); 0 disables reuse
  double skin = 0.25;
  // capacity high-water marks over all workspaces: a pooled workspace that
  // must grow goes straight to the largest size any registration needed
  long long hw_slots = 0, hw_sup = 0;
  // largest candidate radius R_s a grid build has completed at: a new
  // registration at R_s <= hw_radius needs about workspace_estimate() bytes
  // (kreg_register_batch admits registrations against free device memory)
  double hw_radius = 0.0;
  long long mem_budget = 0;  // workspace bytes (kreg_ctx_set_memory_budget; 0 = free device memory)
  long long peak_in_flight = 0, deferred_admissions = 0;
  int chunk_pref = kreg_dev::kPrefChunkUnits;  // sweep chunk size of new lists (kreg_ctx_set_chunk_units)
  long long full_builds = 0, filter_builds = 0;
  // build-stage profile (profiling on): device ms of the build launches,
  // rounds with builds, candidate entries the filters scanned, slots emitted
  double build_ms = 0.0;
  long long build_rounds = 0, filter_entries = 0, built_slots = 0;
  long long full_why[4] = {0, 0, 0, 0};  // grid builds by cause (prepare_build)
  // a resident candidate list is searched again once it holds more than
  // sup_shrink x the entries of a fresh one (its radius^3 ratio; KREG_SUP_SHRINK)
  double sup_shrink = std::getenv("KREG_SUP_SHRINK") ? std::atof(std::getenv("KREG_SUP_SHRINK")) : 3.0;
  long long refilter_builds = 0;         // filter builds that read the resident sweep list
  // sweep-list refilters (opt-in, KREG_REFILTER=1: equal results, but their
  // warp-per-tile kernels are load-imbalanced and measured slower than the
  // candidate-list filter on the KITTI batch)
  bool refilter = std::getenv("KREG_REFILTER") != nullptr;
  kreg_host::Collective collective;  // row-sharded registrations (kreg_ctx_set_collective)
  kreg_host::NcclState* nccl = nullptr;  // kreg_ctx_set_nccl (owned)
  cudaEvent_t timer[2] = {nullptr, nullptr};  // kreg_ctx_timer_mark / _elapsed
  // displacement screen (EvalJob::disp_limit): sweep requests that asked for
  // it, and those whose displacement came from the analytic bound
  long long disp_asked = 0, disp_screened = 0;
  // host-side round accounting (seconds)
  long long rounds = 0;
  double t_prepare = 0.0, t_wait = 0.0, t_total = 0.0;
  double t_build_prep = 0.0, t_sweep_prep = 0.0;
  double t_stage = 0.0, t_upload_issue = 0.0;  // end-to-end calls: host staging, copy issue
  // host <-> device traffic: cloud uploads, results the kernels write into
  // mapped pinned memory (rounds) and explicit copies back
  std::atomic<long long> h2d_bytes{0}, d2h_bytes{0};
  ~kreg_ctx();
};

struct kreg_cloud {
  kreg_ctx* ctx = nullptr;
  int n = 0;
  int dim = 0;
  int fstride = 0;                     // padded device row (floats)
  std::vector<int> chan_off;           // padded channel offsets in a device row
  std::vector<kreg_host::ChannelInfo> schema;
  double diam = 0.0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  kreg_host::DevBuf<double> x, y, z;  // sorted order
  kreg_host::DevBuf<double4> xw;      // sorted order, {x, y, z, 0}
  kreg_host::DevBuf<float> feat;      // sorted order, stride fstride
  std::vector<int> order;              // sorted rank -> original index
  std::vector<int> rank;               // original index -> sorted rank
};

// A pair list plus all device workspace needed to (re)build and sweep it.
// The solver keeps one per registration slot and rebuilds it in place.
struct kreg_pairs {
  kreg_ctx* ctx = nullptr;
  const kreg_cloud* X = nullptr;
  const kreg_cloud* Z = nullptr;
  // reference PairList metadata (inner_product.hpp:18-32)
  double built_at_lengthscale = 0.0;
  double cutoff_radius = 0.0;
  double c_min = 0.0;
  double T_build[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
  long long P = 0;           // valid after the build round completed
  double sigma = 1.0;
  // grid (candidate stage)
  long long n_cells = 0;
  int gx = 0, gy = 0, gz = 0;
  // candidate list: pairs within R_s = cutoff (1 + skin) of Ts z_j with c > c_min
  kreg_host::DevBuf<int4> sup;             // per tile: 32 rows of H_t entries {x_i - Ts z_j, log2 c}
  kreg_host::DevBuf<int> sup_i;            // their target indices
  kreg_host::DevBuf<int> sup_count;
  kreg_host::DevBuf<long long> sup_off;
  bool sup_valid = false;                  // a complete candidate list is resident
  const kreg_cloud* sup_X = nullptr;
  const kreg_cloud* sup_Z = nullptr;
  kreg_dev::CoeffParams sup_cp{};          // coefficient parameters it was built with
  double sup_T[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
  // frame of the sweep-list slots: a slot holds x_i - slot_T z_j (the
  // candidate entry it was filtered from); the sweep subtracts (T - slot_T) z_j
  double slot_T[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
  double sup_radius = 0.0;                 // R_s
  double sup_disp = 0.0;                   // max_j |T_build z_j - sup_T z_j|
  long long sup_entries = 0;
  long long expected_sup = 0;              // capacity hint
  // sweep list
  kreg_host::DevBuf<int> count;            // degree per source (Morton order)
  kreg_host::DevBuf<int> perm, pos, deg_s; // degree-sorted sweep order of the sources
  kreg_host::DevBuf<long long> tile_off;
  kreg_host::DevBuf<int4> slot_buf;        // sweep-list slots {x_i - Ts z_j (FP32 x3), log2 c}
  kreg_host::DevBuf<int> slot_i;           // target index per slot (export only)
  kreg_host::DevBuf<int> unit_off;
  kreg_host::DevBuf<float4> zs;                 // sources in sweep order (FP32)
  kreg_host::DevBuf<kreg_dev::ChunkRec> chunks; // sweep chunk records
  kreg_host::DevBuf<unsigned long long> disp_blk;
  // the previous sweep list while a refilter build reads it (swapped with
  // the buffers above at every refilter build)
  kreg_host::DevBuf<int> alt_perm, alt_pos, alt_deg_s, alt_unit_off;
  kreg_host::DevBuf<long long> alt_tile_off;
  kreg_host::DevBuf<int4> alt_slot_buf;
  kreg_host::DevBuf<float4> alt_zs;
  kreg_host::DevBuf<kreg_dev::ChunkRec> alt_chunks;
  int n_tiles = 0;
  long long slots = 0;                     // valid after the build round
  bool counts_valid = false;               // P / slots known on the host
  double anchor[3] = {0, 0, 0};
  int chunk_pref = kreg_dev::kPrefChunkUnits;  // sweep chunking of this list
  long long expected_pairs = 0;  // capacity hint
  // the last build's request (pairs_export re-runs its emit to recover slot_i)
  kreg_dev::BuildReq last_req{};
  bool index_valid = false;
  // statistics
  long long full_builds = 0, filter_builds = 0;
};

namespace kreg_host {

void set_last_error(const std::string& m);
const char* last_error();

Params to_params(const kreg_kernel_params* p);
void check_kernel_params(const Params& p, const kreg_cloud* schema_of);
void check_same_schema(const kreg_cloud* X, const kreg_cloud* Z, const char* prefix);
std::string describe_schema(const kreg_cloud* c);
void check_config(const kreg_registration_config& c);

kreg_cloud* cloud_create(kreg_ctx* ctx, const kreg_cloud_view* v);
size_t cloud_stage_floats(const kreg_cloud* c);
// PLY file -> device cloud (ply.cu); "property ... skipped" lines appended to warnings
kreg_cloud* cloud_read_ply(kreg_ctx* ctx, const std::string& path, std::string* warnings);
void cloud_download(const kreg_cloud* c, double* xyz, double* features);
// Validation + metadata only (no device copies).
kreg_cloud* cloud_describe(kreg_ctx* ctx, const kreg_cloud_view* v);
// End-to-end batch: clouds (2k, 2k + 1) of job k staged and uploaded by
// worker threads in job order while the solver runs (see ready).
struct AsyncUpload {
  std::vector<std::unique_ptr<kreg_cloud>> clouds;
  std::vector<std::atomic<int>> ready;  // per job: 0 pending, 1 enqueued, -1 failed
  std::vector<cudaEvent_t> done;        // per job: recorded on the context stream after its copies
  std::vector<std::thread> workers;
  std::mutex mu;
  std::exception_ptr error;
  ~AsyncUpload();
};
// `per_unit` consecutive clouds form one unit with one ready flag (2: a
// batch job's X and Z; 1: a sequence frame); `order` (optional, n_units
// entries) is the order in which the workers stage the units
std::unique_ptr<AsyncUpload> cloud_upload_async(kreg_ctx* ctx, const kreg_cloud_view* const* views, int n_units,
                                                int per_unit = 2, std::vector<int> order = {});

// Many clouds: host staging on worker threads, device copies into a context
// arena (valid until the next call of this function on the context).
std::vector<std::unique_ptr<kreg_cloud>> cloud_create_many(kreg_ctx* ctx, const kreg_cloud_view* const* views,
                                                           int n);
double diameter_host(const double* xyz, int n);

// One build request; `pairs` is (re)initialised for X, Z at transform T.
struct BuildJob {
  kreg_pairs* pairs;
  const kreg_cloud* X;
  const kreg_cloud* Z;
  double T[12];
  Params params;       // lengthscale = the build lengthscale
  double cutoff_multiplier;
  double c_min;
  // max_j |T z_j - T_build z_j| against the list being replaced (< 0:
  // unknown); lets the build reuse the resident candidate list
  double disp_hint = -1.0;
  bool force_full = false;
  // end-to-end first builds: the uploads of X / Z (a round on a stream other
  // than the context stream waits for these events, not for every upload)
  cudaEvent_t wait_ev[2] = {nullptr, nullptr};
  bool no_refilter = false;  // filter the candidate list even if the sweep list covers the new one
};

// One evaluation request: M (<= 8) transforms against a built pair list.
struct EvalJob {
  kreg_pairs* pairs;
  int M;
  double T[kreg_dev::kMaxCandidates][12];
  double lengthscale;  // kernel lengthscale of the evaluation
  double sigma = 1.0;  // kernel amplitude of the evaluation (params.sigma, inner_product.cpp:100,126)
  double* out;         // host, M x 8 {F, omega, v, disp}; filled after run_round
  bool grad = true;    // false: F + displacement only (gradient left zero)
  bool second = false; // M = 1: also {dF/d eps, d2F/d eps2} along exp(eps dir) T in out[8..9]
  // > 0: the caller only needs max_j |T_m z_j - T_build z_j| up to this value
  // (solver: the rebuild and reuse thresholds). When an analytic upper bound
  // of every candidate's displacement (bbox of Z) is below it, the sweep runs
  // no displacement items and out[7] receives the bound; the caller's
  // decisions are the same as with the exact maximum.
  double disp_limit = -1.0;
  bool no_disp = false;
  double disp_bound[kreg_dev::kMaxCandidates] = {};
  double dir[6] = {0, 0, 0, 0, 0, 0};
};

// Device resources of one in-flight round.
struct RoundSlot {
  DevBuf<kreg_dev::BuildReq> d_build;
  PinnedBuf<kreg_dev::BuildReq> h_build;
  DevBuf<kreg_dev::SweepReq> d_sweep;
  PinnedBuf<kreg_dev::SweepReq> h_sweep;
  PinnedBuf<double> h_results;             // written by the kernels (mapped pinned memory)
  DevBuf<double> part_arena;                // sweep chunk partials (one slice per request)
  DevBuf<unsigned int> counter_arena;       // sweep chunk counters, self-resetting
  DevBuf<unsigned long long> disp_arena;    // displacement maxima, self-resetting
  // grid searches of the round: cell counts (zero between rounds), cell
  // starts, per-point ints (cell_of, tmp_items, cell_items), cell-ordered
  // positions, scan tiles
  DevBuf<int> g_count, g_start, g_int;
  DevBuf<double> g_pos;
  DevBuf<float> g_feat;
  DevBuf<long long> g_scan;
  cudaEvent_t done = nullptr, ev0 = nullptr, ev1 = nullptr, evb0 = nullptr, evb1 = nullptr;
  // the slot's stream: the context stream, or (slot 1 of a two-group batch)
  // a second stream, so the two groups' rounds overlap on the device (one
  // group's sweep tail with the other's builds and sweep)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ordered = nullptr;  // context-stream work (uploads) before this slot's round
  std::vector<BuildJob> builds;
  std::vector<EvalJob> evals;
  size_t n_res = 0;
  long long sweep_issue = -1;  // index of this round's sweep launch in the context (traces)
  bool in_flight = false;
  ~RoundSlot();
};
RoundSlot* round_slot(kreg_ctx* ctx, int i);

// Executes builds (then, in stream order, evaluations) as batched launches
// and one D2H, without waiting (begin_round); end_round waits for the slot's
// round and stores the results. Builds whose pair list overflowed its
// capacity are grown and re-run transparently. Updates pairs->P.
void begin_round(kreg_ctx* ctx, RoundSlot& S, std::vector<BuildJob>&& builds, std::vector<EvalJob>&& evals);
void end_round(kreg_ctx* ctx, RoundSlot& S);
// begin_round + end_round on the synchronous slot.
void run_round(kreg_ctx* ctx, std::vector<BuildJob>& builds, std::vector<EvalJob>& evals);

double max_point_displacement_dev(kreg_ctx* ctx, const kreg_cloud* Z, const double* built, const double* now);

void pairs_export(kreg_ctx* ctx, const kreg_pairs* p, int64_t* offsets, int32_t* x_index, double* coeff);

// Workspace pool (ctx may be null: plain new/delete).
kreg_pairs* acquire_workspace(kreg_ctx* ctx);
// device bytes a workspace holds; bytes a workspace grown to the context's
// high-water capacities holds
long long workspace_bytes(const kreg_pairs* p);
long long workspace_estimate(const kreg_ctx* ctx);
void release_workspace(kreg_ctx* ctx, kreg_pairs* p);

}  // namespace kreg_host
