/* kreg_b200.h — C-ABI of the B200-native CVO registration engine.
 *
 * Drop-in boundary for the reference's registration hot path
 * (/root/reference/proj, a C++20 library `kreg`). The reference has no FFI;
 * its boundary is the public C++ API. Every entry point below replaces one
 * function of that API (cited per function) with plain pointers, sizes and
 * status codes, so a ctypes / cgo / JNI binding can sit on it directly.
 * include/kreg_b200/kreg.hpp is the C++ RAII layer over this ABI (handles,
 * status -> exception mapping); paper_2012_03683_b200/facade/kreg_facade.cpp
 * restores the reference's own API (names, value types, exceptions) on top
 * of it as a drop-in for inner_product.cpp + registration.cpp.
 *
 * Conventions
 *  - Isometry = double[12], row-major 3x4 [R | t] (reference se3.hpp:27-34).
 *  - Twist    = double[6], (omega, v) (reference se3.hpp:11-21).
 *  - Clouds are uploaded once into device-resident SoA (kreg_cloud); the
 *    reference's PointCloud is immutable after construction
 *    (point_cloud.hpp:48-50), so the handle is too.
 *  - A kreg_ctx is bound to one CUDA device and one stream. It is NOT
 *    thread-safe: the caller serialises calls on one context. Different
 *    contexts may be used concurrently from different host threads.
 *  - Errors: every call returns a kreg_status; the message of the last error
 *    on the calling thread is kreg_last_error(). The codes map back to the
 *    reference's exceptions (errors.hpp:9-36; std::invalid_argument;
 *    std::runtime_error).
 */
#ifndef KREG_B200_H_
#define KREG_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KREG_B200_ABI_VERSION 1

typedef enum {
  KREG_OK = 0,
  KREG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference        */
  KREG_NO_OVERLAP = 2,       /* kreg::NoOverlapError (errors.hpp:25-36)        */
  KREG_CUDA_ERROR = 3,       /* device fault / launch failure                  */
  KREG_OUT_OF_MEMORY = 4,    /* device allocation failed                       */
  KREG_RUNTIME_ERROR = 5,    /* std::runtime_error                             */
  KREG_NO_DEVICE = 6,        /* no CUDA device: there is no CPU fallback       */
  KREG_PARSE_ERROR = 7       /* kreg::ParseError (errors.hpp:9-22)             */
} kreg_status;

/* reference point_cloud.hpp:13 ChannelKind */
typedef enum {
  KREG_KIND_COLOR = 0,
  KREG_KIND_INTENSITY = 1,
  KREG_KIND_SEMANTIC = 2,
  KREG_KIND_CUSTOM = 3
} kreg_channel_kind;

/* reference kernels.hpp:14 KernelForm */
typedef enum { KREG_FORM_SQUARED_EXPONENTIAL = 0, KREG_FORM_LINEAR = 1 } kreg_kernel_form;

/* reference point_cloud.hpp:17-23 Channel */
typedef struct {
  const char* name;
  int32_t dim;
  int32_t kind; /* kreg_channel_kind */
} kreg_channel;

/* Host view of reference PointCloud (point_cloud.hpp:51-76): positions n x 3
 * row-major FP64, features n x dim row-major FP64 (dim = schema total_dim). */
typedef struct {
  const double* xyz;
  int32_t n;
  const double* features; /* may be NULL when dim == 0 */
  int32_t dim;
  const kreg_channel* channels; /* ordered schema; n_channels == 0 => geometric-only */
  int32_t n_channels;
} kreg_cloud_view;

/* reference kernels.hpp:16-20 ChannelParams */
typedef struct {
  double sigma;
  double lengthscale;
  int32_t form; /* kreg_kernel_form */
} kreg_channel_params;

/* reference kernels.hpp:23-33 KernelParams */
typedef struct {
  double sigma;
  double lengthscale;
  const kreg_channel_params* per_channel;
  int32_t n_channels;
} kreg_kernel_params;

/* reference registration.hpp:13-40 RegistrationConfig */
typedef struct {
  double init_lengthscale;
  double subsequent_lengthscale;
  double min_lengthscale;
  double decay_factor;
  int32_t stabilization_window;
  double stabilization_rel_tol;
  int32_t max_iterations;
  double step_init;
  double step_shrink;
  double step_grow;
  int32_t max_backtracks;
  double convergence_twist_norm;
  double cutoff_multiplier;
  double c_min;
} kreg_registration_config;

/* reference registration.hpp:45-60 RegistrationResult. Trace arrays are
 * caller-owned with room for `trace_capacity` entries each (any may be NULL);
 * `iterations` is always the full count, traces are truncated to capacity. */
typedef struct {
  double transform[12];
  int32_t converged;
  int32_t iterations;
  double final_indicator;
  int32_t trace_capacity;
  double* objective_trace;
  double* indicator_trace;
  double* lengthscale_trace;
  double* step_trace;
  double* twist_norm_trace;
  int64_t* pair_count_trace;
  uint8_t* rebuild_trace;
  /* engine statistics (not in the reference): */
  int32_t sweeps;   /* device evaluation passes issued for this registration */
  int32_t rebuilds; /* device pair-list builds */
} kreg_registration_result;

/* reference registration.hpp:85-92 SequenceResult; arrays caller-owned,
 * sized n_frames - 1 (relative, fallback, converged, final_indicator,
 * iterations) and n_frames (trajectory). */
typedef struct {
  double* relative;   /* (n_frames-1) x 12 */
  double* trajectory; /* n_frames x 12 */
  uint8_t* fallback;
  uint8_t* converged;
  double* final_indicator;
  int32_t* iterations;
} kreg_sequence_result;

typedef struct kreg_ctx kreg_ctx;
typedef struct kreg_cloud kreg_cloud;
typedef struct kreg_pairs kreg_pairs;

/* ---------------------------------------------------------------- runtime */
const char* kreg_last_error(void);
int32_t kreg_abi_version(void);
kreg_status kreg_ctx_create(int32_t device, kreg_ctx** out);
kreg_status kreg_ctx_destroy(kreg_ctx* ctx);
kreg_status kreg_ctx_synchronize(kreg_ctx* ctx);
/* Number of device kernels this context has launched so far. */
int64_t kreg_ctx_kernel_launches(const kreg_ctx* ctx);
/* Accumulated device time (ms, CUDA events on the context stream) of the
 * fused sweep kernel and its launch count, for roofline accounting. */
kreg_status kreg_ctx_sweep_stats(const kreg_ctx* ctx, double* sweep_ms, int64_t* sweep_launches,
                                 int64_t* pair_evals);
kreg_status kreg_ctx_set_profiling(kreg_ctx* ctx, int32_t enabled);
/* Device-side timing of a region on the context's stream (CUDA events):
 * mark(0) records the start event, mark(1) the stop event; elapsed returns
 * the milliseconds between them (synchronises on the stop event). Work the
 * context issues from other streams (two-group rounds) is ordered before
 * the stop mark by the calls that issued it (they complete before returning). */
kreg_status kreg_ctx_timer_mark(kreg_ctx* ctx, int32_t which);
/* Displacement screen of the solver's sweeps: {requests that only needed the
 * displacement up to a decision threshold, requests whose displacement came
 * from the analytic bound (no FP64 displacement pass)} since the last reset. */
kreg_status kreg_ctx_screen_stats(const kreg_ctx* ctx, int64_t out[2]);
kreg_status kreg_ctx_timer_elapsed(kreg_ctx* ctx, double* ms);
/* Throughput mode: at most `n` registrations in flight at once (0 = all);
 * a finished registration is replaced by the next one immediately. */
kreg_status kreg_ctx_set_max_active(kreg_ctx* ctx, int32_t n);
/* Device-memory budget of the pair-list workspaces (bytes; 0 = admit against
 * the device's free memory). kreg_register_batch / _sequence start a
 * registration only when its workspace fits; the rest wait for a finished
 * one. Results do not depend on the budget. Engine extension. */
kreg_status kreg_ctx_set_memory_budget(kreg_ctx* ctx, int64_t bytes);
/* Admission since the last reset: {most registrations in flight at once,
 * admissions deferred for memory}. */
kreg_status kreg_ctx_admission_stats(const kreg_ctx* ctx, int64_t out[2]);
/* Host-side round accounting: {rounds, s preparing + launching, s waiting for
 * the device, s preparing builds, s preparing sweeps, s in the solver state
 * machines, device allocations so far (process), s spent in them (process)}. */
kreg_status kreg_ctx_host_stats(const kreg_ctx* ctx, double out[8]);
/* All counters: {sweep kernel ms (profiling on), sweep launches, pair-evals
 * (pairs x candidates), pairs streamed (sum of P per sweep request),
 * sliced-ELL slots streamed, rounds, s preparing, s waiting}. */
kreg_status kreg_ctx_stats(const kreg_ctx* ctx, double out[8]);
kreg_status kreg_ctx_reset_stats(kreg_ctx* ctx);
/* Host <-> device traffic since the last reset: {bytes uploaded (cloud
 * positions FP64 + padded FP32 feature rows), bytes of results the kernels
 * wrote into mapped host memory (per request F, gradient, displacement; per
 * build its status block)}. Engine extension, no reference counterpart. */
kreg_status kreg_ctx_io_stats(const kreg_ctx* ctx, int64_t out[2]);
/* Candidate-list skin: a full build searches the grid at R_s = cutoff (1 +
 * skin) and later builds filter that list while max_j |T z_j - T_s z_j| <=
 * R_s - cutoff (exact: same FP64 predicate); 0 = always search the grid.
 * Default 0.25 (env KREG_SKIN). Engine extension, no reference counterpart. */
kreg_status kreg_ctx_set_candidate_skin(kreg_ctx* ctx, double skin);
/* Sweep chunk size (in 2-step units) of pair lists built from now on:
 * larger chunks amortise per-chunk costs (throughput, default 48), smaller
 * ones spread one list over more warps (single-registration latency).
 * Results are bitwise reproducible for a given setting (env KREG_CHUNK_UNITS).
 * Engine extension, no reference counterpart. */
kreg_status kreg_ctx_set_chunk_units(kreg_ctx* ctx, int32_t units);
/* Builds so far: {grid searches, candidate-list filters}. */
kreg_status kreg_ctx_build_stats(const kreg_ctx* ctx, int64_t out[2]);
/* Build-stage profile since the last reset (needs kreg_ctx_set_profiling):
 * out = {device ms of build launches, rounds with builds, candidate entries
 * scanned by the builds, sweep-list slots emitted, grid builds without a
 * resident candidate list, forced by an overflow or guard, after moving beyond
 * the candidate radius, for other causes, filter builds that read the
 * resident sweep list}. Diagnostic; no reference counterpart. */
kreg_status kreg_ctx_build_profile(const kreg_ctx* ctx, double out[9]);

/* Multi-GPU source-row sharding (configuration C4): every
 * rank registers the replicated target X against its own rows of the source
 * Z, and after every device round the host loop combines the per-rank
 * partial results through this callback: element-wise SUM of `sums` (per
 * request and candidate: F, omega, v; per build: pair count) and MAX of
 * `maxes` (per request and candidate: displacement), in place, identical on
 * all ranks (an all-reduce; NCCL on GPUs). All ranks then make identical
 * decisions, so the replicated loop stays in lockstep. Return 0 on success.
 * NULL clears the hook. */
typedef int32_t (*kreg_collective_fn)(void* user, double* sums, int32_t n_sums, double* maxes, int32_t n_maxes);
kreg_status kreg_ctx_set_collective(kreg_ctx* ctx, kreg_collective_fn fn, void* user);
/* Native NCCL form of the collective (no host callback): every rank creates
 * the communicator from one ncclUniqueId (kreg_nccl_unique_id on rank 0,
 * shared by the caller), then the round's values are combined by NCCL on the
 * context stream. deterministic != 0: one ncclAllGather and a rank-order sum
 * on every rank (bitwise independent of NCCL's algorithm); 0: ncclAllReduce
 * (sum, max). world <= 0 detaches. NCCL is loaded at run time (libnccl.so.2).
 * The deterministic gather is SURVEY.md §8(e)'s "deterministic mode". */
kreg_status kreg_nccl_unique_id(uint8_t id[128]);
kreg_status kreg_ctx_set_nccl(kreg_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t world,
                              int32_t deterministic);
int64_t kreg_ctx_nccl_calls(const kreg_ctx* ctx); /* rounds combined through NCCL */

/* Upload a cloud into device SoA (replaces constructing kreg::PointCloud,
 * point_cloud.cpp:49-59; same validation and messages). */
kreg_status kreg_cloud_create(kreg_ctx* ctx, const kreg_cloud_view* view, kreg_cloud** out);
kreg_status kreg_cloud_destroy(kreg_cloud* cloud);
int32_t kreg_cloud_size(const kreg_cloud* cloud);

/* PLY file straight into a device cloud (replaces read_ply / read_cloud for
 * .ply, cloud_io.cpp:141-297 and cloud_io.hpp:18-26: ascii or
 * binary_little_endian; schema from the properties present; 8/16-bit colour
 * and intensity / 255 / 65535; ParseError -> KREG_PARSE_ERROR with the
 * reference's "path:line: message"). The vertex block is read once into
 * pinned memory, decoded, Morton-ordered and laid out on the device; the cloud
 * is bitwise the one kreg_cloud_create makes from read_ply's PointCloud.
 * `warnings` (may be NULL) receives "property 'name' skipped" lines. */
kreg_status kreg_cloud_read_ply(kreg_ctx* ctx, const char* path, kreg_cloud** out, char* warnings,
                                int32_t warnings_cap);
/* Schema of a device cloud: feature dim and per-channel dims / kinds
 * (arrays of `cap` entries; *n_channels is the full count). */
kreg_status kreg_cloud_schema(const kreg_cloud* cloud, int32_t* dim, int32_t* n_channels, int32_t* dims,
                              int32_t* kinds, int32_t cap);
/* Positions (n x 3 FP64, exact) and features (n x dim, the device's FP32
 * values) back in the original point order; either pointer may be NULL. */
kreg_status kreg_cloud_download(const kreg_cloud* cloud, double* xyz, double* features);

/* --------------------------------------------------- pair engine (L3) */
/* reference inner_product.hpp:50-51 / inner_product.cpp:37-95 build_pairs. */
kreg_status kreg_build_pairs(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z,
                             const double T[12], const kreg_kernel_params* params,
                             double cutoff_multiplier, double c_min, kreg_pairs** out,
                             int64_t* n_pairs);
/* build_pairs again into an existing list (the reference loop's rebuild,
 * registration.cpp:111/126: pairs = build_pairs(X, Z, T, ...)): reuses the
 * list's candidate list when it provably covers the new list (see
 * kreg_ctx_set_candidate_skin), else searches the grid. Same result either way. */
kreg_status kreg_rebuild_pairs(kreg_ctx* ctx, kreg_pairs* pairs, const double T[12],
                               const kreg_kernel_params* params, double cutoff_multiplier,
                               double c_min, int64_t* n_pairs);
kreg_status kreg_pairs_destroy(kreg_pairs* pairs);
int64_t kreg_pairs_size(const kreg_pairs* pairs);
/* Device layout statistics: {pairs, sliced-ELL slots incl. padding, tiles,
 * grid cells}. */
kreg_status kreg_pairs_info(const kreg_pairs* pairs, int64_t out[4]);
/* Copy the pair list out in the reference's layout (inner_product.hpp:18-32):
 * CSR grouped by source j (offsets[n_z+1]), target i ascending inside a group,
 * coeff per entry. Debug / parity path. */
kreg_status kreg_pairs_export(kreg_ctx* ctx, const kreg_pairs* pairs, int64_t* offsets,
                              int32_t* x_index, double* coeff);
/* reference inner_product.hpp:54-55 inner_product. */
kreg_status kreg_inner_product(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X,
                               const kreg_cloud* Z, const double T[12],
                               const kreg_kernel_params* params, double* value);
/* reference inner_product.hpp:67-69 objective_and_gradient:
 * out[0] = F, out[1..3] = grad.omega, out[4..6] = grad.v. */
kreg_status kreg_objective_and_gradient(kreg_ctx* ctx, const kreg_pairs* pairs,
                                        const kreg_cloud* X, const kreg_cloud* Z,
                                        const double T[12], const kreg_kernel_params* params,
                                        double out[7]);
/* Second-order step-size terms along a search direction (north_star item
 * (4); diagnostic only: the reference has no second-order step, SURVEY.md
 * §8 A15, and the engine never uses them for a step decision). For
 * F(eps) = inner_product(pairs, X, Z, exp(eps xi) T) with the pair list held
 * fixed (left perturbation, the reference's candidate form
 * registration.cpp:69), out = {F, dF/d eps, d2F/d eps2} at eps = 0, from one
 * fused device pass (extra per-pair and per-tile reductions of the sweep).
 * The Newton step along xi is -out[1] / out[2] where out[2] < 0. */
kreg_status kreg_directional_terms(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X,
                                   const kreg_cloud* Z, const double T[12], const double xi[6],
                                   const kreg_kernel_params* params, double out[3]);
/* Batched candidate evaluation (the line-search candidates of
 * registration.cpp:63-75 in one device pass): K transforms, out K x 8 =
 * {F, omega[3], v[3], max displacement vs the pair list's build transform}. */
#define KREG_EVAL_GRAD 1u
#define KREG_EVAL_DISP 2u
kreg_status kreg_eval_transforms(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X,
                                 const kreg_cloud* Z, const double* T, int32_t K,
                                 const kreg_kernel_params* params, uint32_t flags, double* out);
/* reference inner_product.hpp:71-75 evaluate_alignment. */
kreg_status kreg_evaluate_alignment(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X,
                                    const kreg_cloud* Z, const double T[12],
                                    const kreg_kernel_params* params, double* value_F,
                                    double* indicator, int64_t* pair_count);
/* reference inner_product.hpp:77-80 indicator (fresh pair list). */
kreg_status kreg_indicator(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z,
                           const double T[12], const kreg_kernel_params* params,
                           double cutoff_multiplier, double c_min, double* value);
/* reference inner_product.cpp:203-236 exact_cosine: dense all-pairs cosine
 * <f_X, f_TZ> / (||f_X|| ||f_Z||) in FP64 on the device (K4, dense.cu);
 * parts (optional) = {cross, ||f_X||^2, ||f_Z||^2}. std::invalid_argument
 * cases map to KREG_INVALID_ARGUMENT (empty clouds, zero-norm functions,
 * schema / params mismatch). Feature rows up to 32 values. */
/* reference eval.cpp:198-235 indicator_sweep (SweepAxis rotation: about z
 * through the centroid; translation: along +x): indicators of `cloud`
 * against perturbed copies at `steps` magnitudes evenly spaced over [0, range]
 * (one magnitude when range == 0). magnitudes / indicators hold max(steps, 1)
 * entries. All pair builds and evaluations run in one batched device round. */
enum { KREG_SWEEP_ROTATION = 0, KREG_SWEEP_TRANSLATION = 1 };
kreg_status kreg_indicator_sweep(kreg_ctx* ctx, const kreg_cloud_view* cloud, const kreg_kernel_params* params,
                                 int32_t axis, double range, int32_t steps, double cutoff_multiplier,
                                 double c_min, double* magnitudes, double* indicators);
/* ---- frame ingest (projection.hpp:12-39, selector.hpp:12-42) */
typedef struct {             /* kreg::CameraIntrinsics (projection.hpp:12-19) */
  double fx, fy, cx, cy;     /* pixels */
  double depth_scale;        /* meters per stored depth unit */
  double max_depth;          /* meters; points beyond are dropped */
  int32_t skip_top_rows;     /* rows excluded from the top of the image */
} kreg_camera_intrinsics;
typedef struct {             /* kreg::SelectorConfig (selector.hpp:12-18) */
  int32_t target_min, target_max;
  double initial_threshold, adjust_factor;
  int32_t max_adjust_rounds;
} kreg_selector_config;
typedef struct {             /* kreg::Selection minus the pixel list (selector.hpp:22-27) */
  int64_t count;             /* selected pixels (rows of the outputs) */
  double threshold;          /* accepted corner threshold */
  int32_t in_band;           /* count landed in [target_min, target_max] */
  int32_t fallback;          /* corner test could not supply target_min: every valid pixel */
  int64_t valid_pixels;      /* pixels with valid depth (the fallback note) */
} kreg_selection_info;
/* select_points (selector.cpp:63-125): rgb w x h x channels (1 or 3),
 * valid_depth w x h mask; writes info->count (u, v) pairs in raster order to
 * pixels_uv when capacity >= info->count (else only info). */
kreg_status kreg_select_points(kreg_ctx* ctx, const uint8_t* rgb, int32_t channels, int32_t width, int32_t height,
                               const uint8_t* valid_depth, const kreg_selector_config* sel, int32_t* pixels_uv,
                               int64_t capacity, kreg_selection_info* info);
/* depth_rgb_to_cloud (projection.cpp:30-75): depth w x h (uint16), rgb w x h x
 * channels, semantics w x h x semantic_channels (float, nullable); writes
 * info->count rows of xyz (3 doubles) and features (3 + semantic_channels
 * doubles: rgb / 255 then the class probabilities) when capacity >=
 * info->count. The pixel test, threshold rounds and back-projection are the
 * reference's, bit for bit. */
kreg_status kreg_depth_rgb_to_cloud(kreg_ctx* ctx, const uint16_t* depth, const uint8_t* rgb, int32_t channels,
                                    const float* semantics, int32_t semantic_channels, int32_t width, int32_t height,
                                    const kreg_camera_intrinsics* intr, const kreg_selector_config* sel, double* xyz,
                                    double* features, int64_t capacity, kreg_selection_info* info);

kreg_status kreg_exact_cosine(kreg_ctx* ctx, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                              const double T[12], const kreg_kernel_params* params, double* cosine,
                              double parts[3]);
/* reference inner_product.hpp:86 max_point_displacement. */
kreg_status kreg_max_point_displacement(kreg_ctx* ctx, const kreg_cloud* Z, const double built[12],
                                        const double now[12], double* value);

/* ------------------------------------------------------- solver (L4) */
/* reference registration.hpp:42 check_config. */
kreg_status kreg_check_config(const kreg_registration_config* config);
/* reference registration.hpp:13-40 defaults. */
void kreg_registration_config_default(kreg_registration_config* config);
/* reference registration.hpp:74-75 anneal_step. */
kreg_status kreg_anneal_step(double lengthscale, const double* history, int32_t n_history,
                             const kreg_registration_config* config, double* next);
/* reference registration.hpp:82-84 line_search. */
kreg_status kreg_line_search(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z,
                             const double T[12], const double g[6],
                             const kreg_kernel_params* params, const kreg_pairs* pairs,
                             const kreg_registration_config* config, double* step);
/* reference registration.hpp:66-68 register_clouds (X = target, Z = source). */
kreg_status kreg_register_clouds(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z,
                                 const double initial[12], const kreg_kernel_params* params,
                                 const kreg_registration_config* config,
                                 kreg_registration_result* result);
/* One rank's share of a row-sharded registration (C4): Z_rows holds this
 * rank's rows of the source, n_z_total the size of the whole source (the
 * indicator denominator sqrt(|X| |Z|), registration.cpp:108-109). Per-round
 * results are combined through the context's collective (kreg_ctx_set_collective);
 * without one this is register_clouds with that denominator. */
kreg_status kreg_register_clouds_rows(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z_rows,
                                      int64_t n_z_total, const double initial[12],
                                      const kreg_kernel_params* params,
                                      const kreg_registration_config* config,
                                      kreg_registration_result* result);
/* Same, from host views: uploads X and Z, registers, frees (end-to-end call). */
kreg_status kreg_register_clouds_host(kreg_ctx* ctx, const kreg_cloud_view* X,
                                      const kreg_cloud_view* Z, const double initial[12],
                                      const kreg_kernel_params* params,
                                      const kreg_registration_config* config,
                                      kreg_registration_result* result);
/* Throughput mode: n independent registrations advanced in lockstep on one
 * device (the reference runs these as an OpenMP loop over trials,
 * eval.cpp:323). statuses[i] receives the per-registration status
 * (KREG_NO_OVERLAP etc.); the call itself fails only on device errors. */
kreg_status kreg_register_batch(kreg_ctx* ctx, int32_t n, const kreg_cloud* const* X,
                                const kreg_cloud* const* Z, const double* initials,
                                const kreg_kernel_params* params,
                                const kreg_registration_config* config,
                                kreg_registration_result* results, int32_t* statuses);
/* End-to-end throughput mode: host views in (uploaded inside the call),
 * results out; same semantics as kreg_register_batch. */
kreg_status kreg_register_batch_host(kreg_ctx* ctx, int32_t n, const kreg_cloud_view* X,
                                     const kreg_cloud_view* Z, const double* initials,
                                     const kreg_kernel_params* params,
                                     const kreg_registration_config* config,
                                     kreg_registration_result* results, int32_t* statuses);
/* reference registration.hpp:99-100 register_sequence. */
kreg_status kreg_register_sequence(kreg_ctx* ctx, const kreg_cloud* const* frames,
                                   int32_t n_frames, const kreg_kernel_params* params,
                                   const kreg_registration_config* config,
                                   kreg_sequence_result* result);
/* Throughput form of register_sequence: frames split into `n_chains`
 * contiguous chains (adjacent chains share one frame), chains registered
 * concurrently in lockstep; chain c covers frames [begin_c, end_c]. The
 * trajectory is composed across chains in order. */
kreg_status kreg_register_sequence_chains(kreg_ctx* ctx, const kreg_cloud* const* frames,
                                          int32_t n_frames, int32_t n_chains,
                                          const kreg_kernel_params* params,
                                          const kreg_registration_config* config,
                                          kreg_sequence_result* result);
/* End-to-end form of kreg_register_sequence_chains (n_chains = 1: exactly
 * kreg_register_sequence): host frames in; they are staged and uploaded on
 * worker threads, in order, while the first pairs already run. The CLI's
 * `kreg sequence` path (main.cpp) after the frames are read. */
kreg_status kreg_register_sequence_host(kreg_ctx* ctx, const kreg_cloud_view* frames,
                                        int32_t n_frames, int32_t n_chains,
                                        const kreg_kernel_params* params,
                                        const kreg_registration_config* config,
                                        kreg_sequence_result* result);
/* Chains with explicit pair spans [begins[s], ends[s]) (pair p registers frames
 * p -> p + 1; spans ordered and disjoint): a rank of a multi-GPU sequence runs
 * its share of the global chain partition. Pairs outside the spans are
 * returned as identity with fallback = 0 and iterations = 0; the trajectory
 * is only meaningful when the spans cover every pair. */
kreg_status kreg_register_sequence_spans(kreg_ctx* ctx, const kreg_cloud* const* frames,
                                         int32_t n_frames, const int32_t* begins, const int32_t* ends,
                                         int32_t n_spans, const kreg_kernel_params* params,
                                         const kreg_registration_config* config,
                                         kreg_sequence_result* result);

/* ------------------------------------------------------- SE(3) host math */
/* reference se3.cpp:48-76 exp, 109-120 compose, 122-127 inverse. */
kreg_status kreg_se3_exp(const double xi[6], double out[12]);
void kreg_se3_compose(const double a[12], const double b[12], double out[12]);
void kreg_se3_inverse(const double T[12], double out[12]);
double kreg_cloud_diameter(const kreg_cloud_view* view); /* point_cloud.cpp:69-87 */

#ifdef __cplusplus
}
#endif

#endif /* KREG_B200_H_ */
