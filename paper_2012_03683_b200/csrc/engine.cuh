// Device-side data layout and kernel entry points of the B200 CVO engine.
//
// Layout in HBM (one registration "slot"; see DESIGN.md §Data layout):
//   Cloud (uploaded once, spatially sorted by a 63-bit Morton key so that
//   index locality == spatial locality):
//     x/y/z        FP64 SoA positions            (build test, q = T z)
//     feat         FP32 rows, stride fstride=4k  (c_ij in the pair build)
//   Grid (per candidate-list build, over target X): dense cell index over
//     the bbox of X, cell = R_s (1 + 1e-7) so the 27-cell stencil is a
//     superset of the FP64 R_s ball; counting sort with a deterministic order
//     inside a cell (ascending point index) -> cell_start[] / cell_items[]
//     plus cell-ordered FP64 positions and FP32 feature rows.
//   Candidate list (reused across levels): per tile of 32 Morton-consecutive
//     sources, 32 rows of H_t entries {x_i - Ts z_j (FP32 x3), log2 c} (16 B)
//     + target index; R_s = cutoff (1 + skin).
//   Sweep list (per build): sources degree-sorted inside windows of 1024,
//     tiles of 32 sorted sources, column height rounded to units of
//     kUnitSteps steps; slot = the candidate entry it was filtered from
//     (16 B, the sweep subtracts (T - Ts) z_j); source-major XOR-swizzled
//     units (slot_index); padding {0,0,0,-inf}; chunk records carry the
//     first tile's sources so the TMA stream has no dependent loads.
//   Sweep scratch: per-chunk and per-group FP64 partials; self-resetting
//     launch control blocks.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace kreg_dev {

constexpr int kSweepThreads = 256;  // threads per persistent sweep CTA (2 CTAs per SM)
#ifndef KREG_SWEEP_CTAS_PER_SM
#define KREG_SWEEP_CTAS_PER_SM 2
#endif
constexpr int kSweepCtasPerSm = KREG_SWEEP_CTAS_PER_SM;  // persistent grid: CTAs per SM
#ifndef KREG_UNIT_STEPS
#define KREG_UNIT_STEPS 2
#endif
#ifndef KREG_SWEEP_STAGES
#define KREG_SWEEP_STAGES 2
#endif
constexpr int kUnitSteps = KREG_UNIT_STEPS;      // degree steps per sweep unit (x 32 lanes x 16 B)
#ifndef KREG_STAGE_UNITS
#define KREG_STAGE_UNITS 4
#endif
constexpr int kStageUnits = KREG_STAGE_UNITS;    // units per TMA stage (4 KB at 2 steps)
constexpr int kSweepStages = KREG_SWEEP_STAGES;  // per-warp TMA ring depth (stages)
#ifndef KREG_MAX_CHUNKS
#define KREG_MAX_CHUNKS 2048
#endif
constexpr int kMaxChunks = KREG_MAX_CHUNKS;      // chunks per request at most (64 groups of 32)
#ifndef KREG_PREF_CHUNK_UNITS
#define KREG_PREF_CHUNK_UNITS 48
#endif
constexpr int kPrefChunkUnits = KREG_PREF_CHUNK_UNITS;  // default preferred chunk size (units)
constexpr int kQueueDepth = 8;                   // chunks a warp may hold in its prefetch queue
#ifndef KREG_MAX_SWEEP_REQS
#define KREG_MAX_SWEEP_REQS 256
#endif
constexpr int kMaxSweepReqs = KREG_MAX_SWEEP_REQS;  // requests per sweep launch (<= kSweepThreads)
constexpr int kChunkGroup = 32;                  // chunk partials summed per group (first reduction level)
constexpr int kMaxChunkGroups = (kMaxChunks + kChunkGroup - 1) / kChunkGroup;
#ifndef KREG_FILTER_WARP
#define KREG_FILTER_WARP 8
#endif
#ifndef KREG_FILTER_THREADS
#define KREG_FILTER_THREADS 128
#endif
constexpr int kFilterWarp = KREG_FILTER_WARP;        // sources per warp of the filter stage
constexpr int kFilterThreads = KREG_FILTER_THREADS;  // threads per filter block
constexpr int kFilterBlock = kFilterThreads / 32 * kFilterWarp;  // sources per filter block (one disp_blk entry)
static_assert(kFilterBlock == 32, "the sweep-list refilter writes one disp_blk entry per 32-source tile");
constexpr int kDispItem = 512;                   // sources per displacement work item
// Sliced-ELL slot of step k of the source in lane l of a tile starting at slot
// tile_off: units of kUnitSteps = 2 steps x 32 sources, source-major inside a
// unit (a source's two slots of a unit share one 32-B sector) with an XOR
// swizzle that keeps the sweep's per-lane LDS.128 conflict-free.
static_assert(KREG_UNIT_STEPS == 2, "slot_index assumes 2-step units");
__host__ __device__ __forceinline__ long long slot_index(long long tile_off, int lane, int k) {
  return tile_off + (long long)(k >> 1) * 64 + 2 * lane + ((k & 1) ^ ((lane >> 2) & 1));
}

constexpr int kMaxChannels = 8;
constexpr int kMaxCandidates = 8;   // candidate transforms per sweep request
constexpr int kOut = 8;             // {F, omega[3], v[3], max displacement}
constexpr int kNvSecond = 11;       // partial values of a second-order request: 7 + {sum w (d.u)^2, u.S, |u|^2 W, (w x u).S}
constexpr int kScanTile = 2048;     // elements per scan tile

struct ChannelDev {
  int offset;     // float offset inside the feature row
  int dim;
  int linear;     // 1 = linear form (dot), 0 = squared exponential
  float kappa;    // SE: -log2(e) / (2 l_c^2)
  float sigma2;   // SE amplitude sigma_c^2 (linear ignores sigma, kernels.cpp:37-42)
};

struct CoeffParams {
  int n_channels;  // 0 => geometric-only (c == 1)
  int fstride;
  float c_min;
  ChannelDev ch[kMaxChannels];
};

// Sweep chunk record (written at build time, TMA-loaded with the chunk's
// first stage): the tile holding the chunk's first unit, the unit where that
// tile ends, and its 32 sources (degree-sorted order) in FP32.
struct alignas(16) ChunkRec {
  int t0;
  int t0_end;
  int pad[2];
  float x[32], y[32], z[32];
};

// One pair-list build for one registration, in two stages:
//  candidate stage (full = 1 only): grid over X + 27-cell search at the
//    enlarged radius R_s = cutoff (1 + skin) around Ts z_j, c_ij and the
//    c > c_min test -> candidate list {x_i - Ts z_j, log2 c} (+ i), 16 B entries;
//  filter stage (always): the reference predicate |x_i - T z_j|^2 <= cutoff^2
//    (inner_product.cpp:69) over the candidate list -> sweep list.
// The filter is exact while max_j |T z_j - Ts z_j| <= R_s - cutoff (triangle
// inequality); the kernel checks that bound and flags the build otherwise.
struct BuildReq {
  const double* xx; const double* xy; const double* xz; const float* xfeat; int n_x;
  const double4* xw;     // X positions as {x, y, z, 0} (filter gathers)
  const double* zx; const double* zy; const double* zz; const float* zfeat; int n_z;
  double T[12];          // build transform, row-major 3x4
  int full;              // run the candidate stage first
  int n_tiles;           // ceil(n_z / 32)
  // candidate stage
  double Ts[12];         // candidate-list transform
  double origin[3];      // grid origin (componentwise min of X)
  double inv_h;          // 1 / cell size
  int gx, gy, gz;        // grid dims
  long long n_cells;
  double sup_cutoff_sq;  // R_s^2
  int* cell_count;       // n_cells (all zero between builds)
  int* cell_start;       // n_cells + 1
  int* cell_of;          // n_x
  int* tmp_items;        // n_x
  int* cell_items;       // n_x
  double* cx; double* cy; double* cz;  // n_x cell-ordered positions
  float* cfeat;          // n_x x fstride cell-ordered feature rows (16-B aligned)
  long long* scan_tiles; // cell-scan workspace (tile sums)
  int* sup_count;        // n_z: candidates of every source
  long long* sup_off;    // n_tiles + 1: candidate tile offsets (entries)
  int4* sup;             // sup_capacity entries {x_i - Ts z_j (FP32 x3), log2 c}
  int* sup_i;            // sup_capacity: their target index i
  long long sup_capacity;
  CoeffParams cp;
  // filter stage
  double cutoff_sq;
  double filter_limit_sq;  // (R_s - cutoff)^2 (minus rounding margin)
  int* count;            // n_z: degree of every source
  int* perm;             // n_z: source at degree-sorted position p
  int* pos;              // n_z: degree-sorted position of source j
  int* deg_s;            // n_z: degree at position p
  long long* tile_off;   // n_tiles + 1: sliced-ELL slot offsets
  int* unit_off;         // n_tiles + 1: sweep work-unit offsets
  float4* zs;            // n_z: sources in degree-sorted order (FP32)
  ChunkRec* chunks;      // kMaxChunks sweep chunk records
  int4* slots;           // capacity slots {x_i - Ts z_j (3 x FP32), log2 c (FP32)}
  int* slot_i;           // capacity: target index i of every slot (export only)
  int write_index;       // emit also writes slot_i (export re-runs the emit with it set)
  long long capacity;
  unsigned long long* disp_blk;   // ceil(n_z / kFilterBlock): per filter block max |T z - Ts z|^2 (bits)
  int chunk_pref;        // sweep chunking of this list (chunk_units)
  // refilter = 1: the filter stage reads the resident sweep list (old_*,
  // built at old_T with a cutoff that covers this one: new pairs are a
  // subset) instead of the candidate list; same predicate on the same
  // entries, so the result equals a candidate-list filter bit for bit
  int refilter;
  double old_T[12];
  const int4* old_slots;
  const int* old_perm;
  const int* old_deg_s;
  const long long* old_tile_off;
  const int* old_unit_off;
  double* status;        // kBuildStatus: {P, slots > cap, slots, cand > cap, cand, |T-Ts| disp, invalid, -}
};
constexpr int kBuildStatus = 8;

// One sweep request: M candidate transforms against one pair list.
struct alignas(16) SweepReq {
  long long units;       // sweep work units when known on the host, else -1
  const long long* tile_off;
  const int* unit_off;
  const float4* zs;      // sources in degree-sorted order (FP32)
  const ChunkRec* chunks;
  int n_tiles;
  const int4* slots;
  long long capacity;    // slot capacity (an overflowed build is skipped)
  int grad;              // 0: F (+ displacement) only, 1: F + gradient
  int no_disp;           // 1: no displacement items (the host's bound decides, EvalJob::disp_limit)
  int second;            // 1 (M = 1, grad): also dF/d eps, d2F/d eps2 along exp(eps xi) T -> out[kOut .. kOut + 1]
  float dir[6];          // xi = {omega, omega x anchor + v} (second-order requests)
  int chunk_pref;        // the list's sweep chunking (chunk_units)
  const double* zx; const double* zy; const double* zz;  // source, sorted
  int n_z;
  int M;
  double T[kMaxCandidates][12];
  double Tb[12];         // pair-list build transform (displacement reference)
  float Td[kMaxCandidates][12];  // {R_m - R_s, t_m - t_s}: (T_m - T_s) z, T_s the slots' frame
  float Ta[kMaxCandidates][12];  // {R_m, t_m - anchor}: T_m z - anchor (torque arm)
  double anchor[3];
  float kappa;           // -log2(e) / (2 l^2): ex2 argument per m^2
  double sigma2;
  double inv_l2;
  double* partials;      // (kMaxChunks + kMaxChunkGroups) x M x (7 | 1): chunk, then group partials
  unsigned long long* disp_bits;  // M, max squared displacement (self-resetting)
  double* out;           // M x kOut
};

// Once per device (kreg_ctx_create): kernel attributes of the current device.
cudaError_t init_device();

// All launches go to `stream`; d_reqs are device copies of h_reqs.
void build_pairs_batched(const BuildReq* h_reqs, const BuildReq* d_reqs, int n, cudaStream_t stream);
// d_ctl: sweep_ctl_bytes(n) bytes of launch control blocks, zero between
// launches (the kernels reset them).
size_t sweep_ctl_bytes(int n);
void sweep_batched(const SweepReq* h_reqs, const SweepReq* d_reqs, int n, int sm_count, unsigned* d_ctl,
                   cudaStream_t stream, cudaEvent_t sweep_begin, cudaEvent_t sweep_end);
void displacement(const double* zx, const double* zy, const double* zz, int n, const double* d_T2,
                  unsigned long long* d_out, cudaStream_t stream);

// Frame ingest (ingest.cu): depth + RGB -> FAST-selected pixels -> cloud rows.
struct IngestReq {
  int w, h, channels, sem_channels;
  const uint16_t* depth;     // w x h (null for select_points)
  const uint8_t* rgb;        // w x h x channels
  const float* sem;          // w x h x sem_channels or null
  const uint8_t* valid_in;   // w x h mask (select_points) or null: derived from depth
  int skip_top_rows;
  double depth_scale, max_depth, fx, fy, cx, cy;
  uint8_t* score;            // w x h: FAST score clamped at 0
  uint8_t* valid;            // w x h
  unsigned long long* hist;  // 256 bins of the score over valid pixels
  double threshold;          // selection: score > threshold (or every valid pixel)
  int fallback;
  int* block_count;          // per 1024-pixel block
  long long* block_off;      // exclusive prefix (+ total)
  long long cap;             // output rows
  int* pixels;               // cap x (u, v)
  double* xyz;               // cap x 3 or null
  double* feat;              // cap x (3 + sem_channels)
};
void ingest_score(const IngestReq& R, cudaStream_t stream);
int ingest_blocks(long long pixels);
void ingest_emit(const IngestReq& R, bool count_only, cudaStream_t stream);

// K4 dense double sum over all pairs (a, b) of two clouds (dense.cu).
constexpr int kMaxDenseDim = 32;
struct DenseChannel {
  int offset, dim, linear;
  double neg_inv_2l2;  // SE: -1 / (2 l_k^2)
};
struct DenseReq {
  const double* a;   // n_a x 3 positions
  const double* af;  // n_a x D features
  const double* b;   // n_b x 3 positions (already transformed)
  const double* bf;  // n_b x D features
  int n_a, n_b, D;
  int n_channels;
  DenseChannel ch[kMaxChannels];
  double neg_inv_2l2;  // geometric -1 / (2 l^2)
  double pref;         // sigma^2 x prod over SE channels sigma_k^2
  double* partials;    // dense_blocks_a(max n_a) x b_chunks
};
void dense_sums(const DenseReq* h_reqs, const DenseReq* d_reqs, int n, int b_chunks, cudaStream_t stream);
int dense_blocks_a(int n_a);

// Re-run a list's emit pass with write_index set (pairs_export).
void filter_emit_index(const BuildReq* d_req, int n_z, cudaStream_t stream);
void interleave_positions(const double* x, const double* y, const double* z, int n, double4* out, cudaStream_t stream);

long long kernel_launch_count();
void note_launches(int n);  // launches issued from other translation units

}  // namespace kreg_dev
