// C-ABI of the B200 CVO engine (include/kreg_b200.h). Every entry point maps
// C++ exceptions to kreg_status + a thread-local message; there is no CPU
// fallback: without a CUDA device every compute entry point fails with
// KREG_NO_DEVICE / KREG_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

#include "../../include/kreg_b200.h"
#include "engine_host.hpp"
#include "se3_host.hpp"
#include "solver.hpp"

using namespace kreg_host;

namespace {

template <typename Fn>
kreg_status guarded(Fn&& fn) {
  try {
    fn();
    return KREG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return KREG_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return KREG_RUNTIME_ERROR;
  }
}

void require(bool ok, const char* what) {
  if (!ok) throw Error(KREG_INVALID_ARGUMENT, what);
}

void check_build_args(const kreg_cloud* X, const kreg_cloud* Z, const Params& p, double cutoff_multiplier,
                      double c_min) {
  // inner_product.cpp:39-46
  check_same_schema(X, Z, "");
  check_kernel_params(p, X);
  if (!(cutoff_multiplier >= 1.0)) throw Error(KREG_INVALID_ARGUMENT, "build_pairs: cutoff_multiplier must be >= 1");
  if (c_min < 0.0 || c_min >= 1.0) throw Error(KREG_INVALID_ARGUMENT, "build_pairs: c_min must lie in [0, 1)");
}

// Evaluate K transforms (any K) against a built pair list; out K x 8.
void eval_many(kreg_ctx* ctx, kreg_pairs* p, const double* T, int K, double lengthscale, double sigma, double* out) {
  std::vector<BuildJob> none;
  std::vector<EvalJob> evals;
  for (int b = 0; b < K; b += kreg_dev::kMaxCandidates) {
    EvalJob e;
    e.pairs = p;
    e.M = std::min(kreg_dev::kMaxCandidates, K - b);
    for (int m = 0; m < e.M; ++m) std::memcpy(e.T[m], T + 12 * (b + m), sizeof(double) * 12);
    e.lengthscale = lengthscale;
    e.sigma = sigma;
    e.out = out + static_cast<size_t>(b) * kreg_dev::kOut;
    evals.push_back(e);
  }
  run_round(ctx, none, evals);
}

kreg_pairs* build(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z, const double* T, const Params& p,
                  double cutoff_multiplier, double c_min) {
  check_build_args(X, Z, p, cutoff_multiplier, c_min);
  auto pr = std::make_unique<kreg_pairs>();
  pr->ctx = ctx;
  pr->X = X;
  pr->Z = Z;
  pr->built_at_lengthscale = p.lengthscale;
  pr->cutoff_radius = cutoff_multiplier * p.lengthscale;
  pr->c_min = c_min;
  pr->sigma = p.sigma;
  std::memcpy(pr->T_build, T, sizeof(double) * 12);
  pr->P = 0;
  if (X->n > 0 && Z->n > 0) {  // inner_product.cpp:55-56: empty clouds => empty list
    std::vector<BuildJob> builds(1);
    builds[0].pairs = pr.get();
    builds[0].X = X;
    builds[0].Z = Z;
    std::memcpy(builds[0].T, T, sizeof(double) * 12);
    builds[0].params = p;
    builds[0].cutoff_multiplier = cutoff_multiplier;
    builds[0].c_min = c_min;
    std::vector<EvalJob> none;
    run_round(ctx, builds, none);
  }
  return pr.release();
}

void check_pairs_match(const kreg_pairs* p, const kreg_cloud* X, const kreg_cloud* Z) {
  require(p != nullptr, "pairs must not be NULL");
  require(p->X == X && p->Z == Z, "pair list was built for different clouds");
}

void fill_sequence(const std::vector<double>& rel, const std::vector<uint8_t>& fb, const std::vector<uint8_t>& cv,
                   const std::vector<double>& fi, const std::vector<int>& it, kreg_sequence_result* out) {
  const size_t m = fb.size();
  double traj[12];
  kreg_se3::identity(traj);
  std::memcpy(out->trajectory, traj, sizeof(traj));
  for (size_t k = 0; k < m; ++k) {
    std::memcpy(out->relative + 12 * k, rel.data() + 12 * k, sizeof(double) * 12);
    out->fallback[k] = fb[k];
    out->converged[k] = cv[k];
    out->final_indicator[k] = fi[k];
    out->iterations[k] = it[k];
    double next[12];
    kreg_se3::compose(traj, rel.data() + 12 * k, next);  // registration.cpp:226
    std::memcpy(traj, next, sizeof(traj));
    std::memcpy(out->trajectory + 12 * (k + 1), traj, sizeof(traj));
  }
}

// Registers the chains [begin_c, end_c] of `frames` concurrently. Inside a
// chain, pair k starts from the previous relative motion at the subsequent
// lengthscale (registration.cpp:191-230); NoOverlapError => fallback. Every
// pair of every chain is one job of one lockstep batch; a chain's next pair
// joins the batch the moment its predecessor finishes (no barrier across
// chains). A chain's first pair starts from identity at init_lengthscale, as
// register_sequence's first pair does: chains are independent sequences
// (SURVEY.md 8(d) C5), so a span that starts mid-sequence does not inherit the
// motion of the pair before it (the single-chain call is exactly the
// reference's register_sequence).
void run_chains(kreg_ctx* ctx, const kreg_cloud* const* frames, int n_frames, const std::vector<int>& begins,
                const std::vector<int>& ends, const Params& params, const kreg_registration_config& config,
                kreg_sequence_result* out, const std::atomic<int>* frame_ready = nullptr,
                const cudaEvent_t* frame_done = nullptr) {
  const int m = n_frames - 1;
  std::vector<double> rel(static_cast<size_t>(m) * 12);
  for (int k = 0; k < m; ++k) kreg_se3::identity(rel.data() + 12 * k);  // pairs outside the spans
  std::vector<uint8_t> fb(static_cast<size_t>(m)), cv(static_cast<size_t>(m));
  std::vector<double> fi(static_cast<size_t>(m));
  std::vector<int> it(static_cast<size_t>(m));
  const int nc = static_cast<int>(begins.size());
  // jobs ordered chain head first (all heads start at once), then by position
  std::vector<int> pair_of;
  std::vector<RegJob> jobs;
  for (int pos = 0;; ++pos) {
    bool any = false;
    for (int c = 0; c < nc; ++c) {
      const int k = begins[c] + pos + 1;  // pair (k-1, k)
      if (k > ends[c]) continue;
      any = true;
      RegJob j;
      j.X = frames[k - 1];
      j.Z = frames[k];
      if (frame_ready) {  // end-to-end: the pair starts once both frames are on the device
        j.ready = &frame_ready[k - 1];
        j.ready2 = &frame_ready[k];
        if (frame_done) {
          j.ready_ev = frame_done[k - 1];
          j.ready_ev2 = frame_done[k];
        }
      }
      kreg_se3::identity(j.initial);
      j.params = params;
      j.cfg = config;
      if (pos > 0) j.cfg.init_lengthscale = config.subsequent_lengthscale;
      j.cfg.min_lengthscale = std::min(j.cfg.min_lengthscale, j.cfg.init_lengthscale);
      jobs.push_back(j);
      pair_of.push_back(k - 1);
    }
    if (!any) break;
  }
  std::vector<int> job_of_pair(static_cast<size_t>(m), -1);
  for (size_t q = 0; q < jobs.size(); ++q) job_of_pair[static_cast<size_t>(pair_of[q])] = static_cast<int>(q);
  for (size_t q = 0; q < jobs.size(); ++q) {
    const int p = pair_of[q];
    const bool head = std::find(begins.begin(), begins.end(), p) != begins.end();
    if (!head && p > 0 && job_of_pair[static_cast<size_t>(p - 1)] >= 0) {
      jobs[q].pred = job_of_pair[static_cast<size_t>(p - 1)];
      jobs[static_cast<size_t>(jobs[q].pred)].succ = static_cast<int>(q);
    }
  }
  std::vector<kreg_registration_result> results(jobs.size());
  for (size_t q = 0; q < jobs.size(); ++q) {
    std::memset(&results[q], 0, sizeof(kreg_registration_result));
    jobs[q].out = &results[q];
  }
  register_many(ctx, jobs);
  for (size_t q = 0; q < jobs.size(); ++q) {
    const int slot = pair_of[q];
    const RegJob& j = jobs[q];
    if (j.status == KREG_OK) {
      std::memcpy(rel.data() + 12 * slot, results[q].transform, sizeof(double) * 12);
      fb[slot] = 0;
      cv[slot] = results[q].converged ? 1 : 0;
      fi[slot] = results[q].final_indicator;
      it[slot] = results[q].iterations;
    } else if (j.status == KREG_NO_OVERLAP) {
      std::memcpy(rel.data() + 12 * slot, j.initial, sizeof(double) * 12);  // the previous relative motion
      fb[slot] = 1;
      cv[slot] = 0;
      fi[slot] = 0.0;
      it[slot] = 0;
    } else {
      throw Error(j.status, j.error);
    }
  }
  fill_sequence(rel, fb, cv, fi, it, out);
}

}  // namespace

extern "C" {

const char* kreg_last_error(void) { return last_error(); }
int32_t kreg_abi_version(void) { return KREG_B200_ABI_VERSION; }

kreg_status kreg_ctx_create(int32_t device, kreg_ctx** out) {
  return guarded([&] {
    require(out != nullptr, "out must not be NULL");
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw Error(KREG_NO_DEVICE, "no CUDA device available (the engine has no CPU fallback)");
    }
    require(device >= 0 && device < n, "device index out of range");
    auto ctx = std::make_unique<kreg_ctx>();
    ctx->device = device;
    KREG_CUDA(cudaSetDevice(device));
    KREG_CUDA(kreg_dev::init_device());
    KREG_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
    KREG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->launches_base = kreg_dev::kernel_launch_count();
    if (const char* sk = std::getenv("KREG_SKIN")) ctx->skin = std::atof(sk);
    if (const char* cu = std::getenv("KREG_CHUNK_UNITS")) ctx->chunk_pref = std::max(1, std::atoi(cu));
    *out = ctx.release();
  });
}

kreg_status kreg_ctx_set_chunk_units(kreg_ctx* ctx, int32_t units) {
  return guarded([&] {
    require(ctx != nullptr, "ctx must not be NULL");
    require(units >= 1 && units <= 4096, "chunk units must lie in [1, 4096]");
    ctx->chunk_pref = units;
  });
}

kreg_status kreg_ctx_set_candidate_skin(kreg_ctx* ctx, double skin) {
  return guarded([&] {
    require(ctx != nullptr, "ctx must not be NULL");
    require(skin >= 0.0 && skin <= 4.0, "candidate skin must lie in [0, 4]");
    ctx->skin = skin;
  });
}

kreg_status kreg_ctx_build_stats(const kreg_ctx* ctx, int64_t out[2]) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, "NULL argument");
    out[0] = ctx->full_builds;
    out[1] = ctx->filter_builds;
  });
}

kreg_status kreg_ctx_build_profile(const kreg_ctx* ctx, double out[9]) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, "NULL argument");
    out[0] = ctx->build_ms;
    out[1] = static_cast<double>(ctx->build_rounds);
    out[2] = static_cast<double>(ctx->filter_entries);
    out[3] = static_cast<double>(ctx->built_slots);
    for (int k = 0; k < 4; ++k) out[4 + k] = static_cast<double>(ctx->full_why[k]);
    out[8] = static_cast<double>(ctx->refilter_builds);
  });
}

kreg_status kreg_ctx_destroy(kreg_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->d_T2.release();
    ctx->d_disp.release();
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

kreg_status kreg_ctx_synchronize(kreg_ctx* ctx) {
  return guarded([&] { KREG_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int64_t kreg_ctx_kernel_launches(const kreg_ctx* ctx) { return kreg_dev::kernel_launch_count() - ctx->launches_base; }

kreg_status kreg_ctx_sweep_stats(const kreg_ctx* ctx, double* sweep_ms, int64_t* sweep_launches, int64_t* pair_evals) {
  return guarded([&] {
    if (sweep_ms) *sweep_ms = ctx->sweep_ms;
    if (sweep_launches) *sweep_launches = ctx->sweep_launches;
    if (pair_evals) *pair_evals = ctx->pair_evals;
  });
}

kreg_status kreg_ctx_host_stats(const kreg_ctx* ctx, double out[8]) {
  return guarded([&] {
    out[0] = static_cast<double>(ctx->rounds);
    out[1] = ctx->t_prepare;
    out[2] = ctx->t_wait;
    out[3] = ctx->t_build_prep;
    out[4] = ctx->t_sweep_prep;
    out[5] = ctx->t_total;
    out[6] = static_cast<double>(g_device_allocs);
    out[7] = g_device_alloc_seconds;
    if (ctx->t_stage > 0.0) out[4] = ctx->t_stage;  // end-to-end runs: host staging replaces sweep prep
  });
}

kreg_status kreg_ctx_stats(const kreg_ctx* ctx, double out[8]) {
  return guarded([&] {
    out[0] = ctx->sweep_ms;
    out[1] = static_cast<double>(ctx->sweep_launches);
    out[2] = static_cast<double>(ctx->pair_evals);
    out[3] = static_cast<double>(ctx->pairs_streamed);
    out[4] = static_cast<double>(ctx->slots_streamed);
    out[5] = static_cast<double>(ctx->rounds);
    out[6] = ctx->t_prepare;
    out[7] = ctx->t_wait;
  });
}

kreg_status kreg_ctx_screen_stats(const kreg_ctx* ctx, int64_t out[2]) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, "NULL argument");
    out[0] = ctx->disp_asked;
    out[1] = ctx->disp_screened;
  });
}

kreg_status kreg_ctx_io_stats(const kreg_ctx* ctx, int64_t out[2]) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, "NULL argument");
    out[0] = ctx->h2d_bytes.load();
    out[1] = ctx->d2h_bytes.load();
  });
}

kreg_status kreg_ctx_set_max_active(kreg_ctx* ctx, int32_t n) {
  return guarded([&] {
    require(ctx != nullptr && n >= 0, "invalid argument");
    ctx->max_active = n;
  });
}

kreg_status kreg_ctx_set_memory_budget(kreg_ctx* ctx, int64_t bytes) {
  return guarded([&] {
    require(ctx != nullptr && bytes >= 0, "invalid argument");
    ctx->mem_budget = bytes;
  });
}

kreg_status kreg_ctx_admission_stats(const kreg_ctx* ctx, int64_t out[2]) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, "NULL argument");
    out[0] = ctx->peak_in_flight;
    out[1] = ctx->deferred_admissions;
  });
}

kreg_status kreg_ctx_set_profiling(kreg_ctx* ctx, int32_t enabled) {
  return guarded([&] { ctx->profiling = enabled != 0; });
}

kreg_status kreg_ctx_reset_stats(kreg_ctx* ctx) {
  return guarded([&] {
    ctx->sweep_ms = 0.0;
    ctx->sweep_launches = 0;
    ctx->pair_evals = 0;
    ctx->pairs_streamed = 0;
    ctx->slots_streamed = 0;
    ctx->rounds = 0;
    ctx->t_prepare = ctx->t_wait = ctx->t_total = 0.0;
    ctx->t_build_prep = ctx->t_sweep_prep = 0.0;
    ctx->t_stage = ctx->t_upload_issue = 0.0;
    ctx->h2d_bytes = 0;
    ctx->d2h_bytes = 0;
    ctx->peak_in_flight = 0;
    ctx->deferred_admissions = 0;
    ctx->launches_base = kreg_dev::kernel_launch_count();
    ctx->full_builds = ctx->filter_builds = 0;
    ctx->build_ms = 0.0;
    ctx->build_rounds = ctx->filter_entries = ctx->built_slots = 0;
    ctx->disp_asked = ctx->disp_screened = 0;
    for (long long& w : ctx->full_why) w = 0;
    ctx->refilter_builds = 0;
  });
}

kreg_status kreg_cloud_create(kreg_ctx* ctx, const kreg_cloud_view* view, kreg_cloud** out) {
  return guarded([&] {
    require(ctx && view && out, "NULL argument");
    *out = cloud_create(ctx, view);
  });
}

kreg_status kreg_cloud_destroy(kreg_cloud* cloud) {
  return guarded([&] { delete cloud; });
}

int32_t kreg_cloud_size(const kreg_cloud* cloud) { return cloud ? cloud->n : 0; }

kreg_status kreg_cloud_read_ply(kreg_ctx* ctx, const char* path, kreg_cloud** out, char* warnings,
                                int32_t warnings_cap) {
  return guarded([&] {
    require(ctx && path && out, "NULL argument");
    std::string w;
    *out = cloud_read_ply(ctx, path, &w);
    if (warnings && warnings_cap > 0) {
      const size_t k = std::min(w.size(), static_cast<size_t>(warnings_cap - 1));
      std::memcpy(warnings, w.data(), k);
      warnings[k] = '\0';
    }
  });
}

kreg_status kreg_cloud_schema(const kreg_cloud* cloud, int32_t* dim, int32_t* n_channels, int32_t* dims,
                              int32_t* kinds, int32_t cap) {
  return guarded([&] {
    require(cloud != nullptr, "NULL argument");
    if (dim) *dim = cloud->dim;
    if (n_channels) *n_channels = static_cast<int32_t>(cloud->schema.size());
    for (size_t k = 0; k < cloud->schema.size() && static_cast<int32_t>(k) < cap; ++k) {
      if (dims) dims[k] = cloud->schema[k].dim;
      if (kinds) kinds[k] = cloud->schema[k].kind;
    }
  });
}

kreg_status kreg_cloud_download(const kreg_cloud* cloud, double* xyz, double* features) {
  return guarded([&] {
    require(cloud != nullptr, "NULL argument");
    cloud_download(cloud, xyz, features);
  });
}

kreg_status kreg_build_pairs(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z, const double T[12],
                             const kreg_kernel_params* params, double cutoff_multiplier, double c_min,
                             kreg_pairs** out, int64_t* n_pairs) {
  return guarded([&] {
    require(ctx && X && Z && T && params && out, "NULL argument");
    kreg_pairs* p = build(ctx, X, Z, T, to_params(params), cutoff_multiplier, c_min);
    *out = p;
    if (n_pairs) *n_pairs = p->P;
  });
}

kreg_status kreg_rebuild_pairs(kreg_ctx* ctx, kreg_pairs* pairs, const double T[12],
                               const kreg_kernel_params* params, double cutoff_multiplier, double c_min,
                               int64_t* n_pairs) {
  return guarded([&] {
    require(ctx && pairs && T && params, "NULL argument");
    require(pairs->X && pairs->Z, "pair list has no clouds");
    const Params p = to_params(params);
    check_build_args(pairs->X, pairs->Z, p, cutoff_multiplier, c_min);
    if (pairs->X->n > 0 && pairs->Z->n > 0) {
      std::vector<BuildJob> builds(1);
      builds[0].pairs = pairs;
      builds[0].X = pairs->X;
      builds[0].Z = pairs->Z;
      std::memcpy(builds[0].T, T, sizeof(double) * 12);
      builds[0].params = p;
      builds[0].cutoff_multiplier = cutoff_multiplier;
      builds[0].c_min = c_min;
      builds[0].disp_hint =
          pairs->counts_valid ? max_point_displacement_dev(ctx, pairs->Z, pairs->T_build, T) : -1.0;
      std::vector<EvalJob> none;
      run_round(ctx, builds, none);
    } else {
      pairs->built_at_lengthscale = p.lengthscale;
      pairs->cutoff_radius = cutoff_multiplier * p.lengthscale;
      std::memcpy(pairs->T_build, T, sizeof(double) * 12);
      pairs->P = 0;
    }
    if (n_pairs) *n_pairs = pairs->P;
  });
}

kreg_status kreg_pairs_destroy(kreg_pairs* pairs) {
  return guarded([&] { delete pairs; });
}

int64_t kreg_pairs_size(const kreg_pairs* pairs) { return pairs ? pairs->P : 0; }

kreg_status kreg_pairs_info(const kreg_pairs* pairs, int64_t out[4]) {
  return guarded([&] {
    require(pairs && out, "NULL argument");
    out[0] = pairs->P;
    out[1] = pairs->slots;
    out[2] = pairs->n_tiles;
    out[3] = pairs->n_cells;
  });
}

kreg_status kreg_pairs_export(kreg_ctx* ctx, const kreg_pairs* pairs, int64_t* offsets, int32_t* x_index,
                              double* coeff) {
  return guarded([&] {
    require(ctx && pairs && offsets, "NULL argument");
    if (!pairs->Z || pairs->Z->n == 0 || pairs->P == 0) {
      const int nz = pairs->Z ? pairs->Z->n : 0;
      for (int j = 0; j <= nz; ++j) offsets[j] = 0;
      return;
    }
    pairs_export(ctx, pairs, offsets, x_index, coeff);
  });
}

kreg_status kreg_eval_transforms(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X, const kreg_cloud* Z,
                                 const double* T, int32_t K, const kreg_kernel_params* params, uint32_t flags,
                                 double* out) {
  (void)flags;  // gradient and displacement are always produced by the fused sweep
  return guarded([&] {
    require(ctx && pairs && T && params && out && K >= 0, "invalid argument");
    check_pairs_match(pairs, X, Z);
    if (K == 0) return;
    if (pairs->P == 0) {
      // inner_product.cpp:98 / :124: empty list => zeros (displacement still defined)
      for (int k = 0; k < K; ++k) {
        std::memset(out + 8 * k, 0, sizeof(double) * 8);
        out[8 * k + 7] = max_point_displacement_dev(ctx, Z, pairs->T_build, T + 12 * k);
      }
      return;
    }
    eval_many(ctx, const_cast<kreg_pairs*>(pairs), T, K, params->lengthscale, params->sigma, out);
  });
}

kreg_status kreg_directional_terms(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X, const kreg_cloud* Z,
                                   const double T[12], const double xi[6], const kreg_kernel_params* params,
                                   double out[3]) {
  return guarded([&] {
    require(ctx && pairs && T && xi && params && out, "invalid argument");
    check_pairs_match(pairs, X, Z);
    if (pairs->P == 0) {  // empty list: F and its derivatives vanish
      out[0] = out[1] = out[2] = 0.0;
      return;
    }
    double o[kreg_dev::kOut + 2];
    std::vector<BuildJob> none;
    std::vector<EvalJob> evals(1);
    EvalJob& e = evals[0];
    e.pairs = const_cast<kreg_pairs*>(pairs);
    e.M = 1;
    std::memcpy(e.T[0], T, sizeof(double) * 12);
    e.lengthscale = params->lengthscale;
    e.sigma = params->sigma;
    e.out = o;
    e.second = true;
    std::memcpy(e.dir, xi, sizeof(e.dir));
    run_round(ctx, none, evals);
    out[0] = o[0];
    out[1] = o[kreg_dev::kOut];
    out[2] = o[kreg_dev::kOut + 1];
  });
}

kreg_status kreg_inner_product(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X, const kreg_cloud* Z,
                               const double T[12], const kreg_kernel_params* params, double* value) {
  double o[8];
  const kreg_status s = kreg_eval_transforms(ctx, pairs, X, Z, T, 1, params, 0, o);
  if (s == KREG_OK) *value = o[0];
  return s;
}

kreg_status kreg_objective_and_gradient(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X,
                                        const kreg_cloud* Z, const double T[12], const kreg_kernel_params* params,
                                        double out[7]) {
  double o[8];
  const kreg_status s = kreg_eval_transforms(ctx, pairs, X, Z, T, 1, params, KREG_EVAL_GRAD, o);
  if (s == KREG_OK) std::memcpy(out, o, sizeof(double) * 7);
  return s;
}

kreg_status kreg_evaluate_alignment(kreg_ctx* ctx, const kreg_pairs* pairs, const kreg_cloud* X, const kreg_cloud* Z,
                                    const double T[12], const kreg_kernel_params* params, double* value_F,
                                    double* indicator, int64_t* pair_count) {
  double o[8];
  const kreg_status s = kreg_eval_transforms(ctx, pairs, X, Z, T, 1, params, 0, o);
  if (s != KREG_OK) return s;
  // inner_product.cpp:159-168
  const double denom = std::sqrt(static_cast<double>(X->n) * static_cast<double>(Z->n));
  if (value_F) *value_F = o[0];
  if (indicator) *indicator = denom > 0.0 ? o[0] / denom : 0.0;
  if (pair_count) *pair_count = pairs->P;
  return KREG_OK;
}

kreg_status kreg_indicator(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z, const double T[12],
                           const kreg_kernel_params* params, double cutoff_multiplier, double c_min, double* value) {
  return guarded([&] {
    require(ctx && X && Z && T && params && value, "NULL argument");
    // inner_product.cpp:170-177
    if (X->n == 0 || Z->n == 0) throw Error(KREG_INVALID_ARGUMENT, "indicator: clouds must be non-empty");
    std::unique_ptr<kreg_pairs> p(build(ctx, X, Z, T, to_params(params), cutoff_multiplier, c_min));
    double o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (p->P > 0) eval_many(ctx, p.get(), T, 1, params->lengthscale, params->sigma, o);
    const double denom = std::sqrt(static_cast<double>(X->n) * static_cast<double>(Z->n));
    *value = denom > 0.0 ? o[0] / denom : 0.0;
  });
}

kreg_status kreg_max_point_displacement(kreg_ctx* ctx, const kreg_cloud* Z, const double built[12],
                                        const double now[12], double* value) {
  return guarded([&] {
    require(ctx && Z && built && now && value, "NULL argument");
    *value = max_point_displacement_dev(ctx, Z, built, now);
  });
}

kreg_status kreg_check_config(const kreg_registration_config* config) {
  return guarded([&] { check_config(*config); });
}

void kreg_registration_config_default(kreg_registration_config* c) {
  // registration.hpp:18-39
  c->init_lengthscale = 0.95;
  c->subsequent_lengthscale = 0.1;
  c->min_lengthscale = 0.0475;
  c->decay_factor = 0.98;
  c->stabilization_window = 5;
  c->stabilization_rel_tol = 1e-5;
  c->max_iterations = 2000;
  c->step_init = 0.1;
  c->step_shrink = 0.5;
  c->step_grow = 1.2;
  c->max_backtracks = 20;
  c->convergence_twist_norm = 1e-5;
  c->cutoff_multiplier = 3.0;
  c->c_min = 1e-4;
}

kreg_status kreg_anneal_step(double lengthscale, const double* history, int32_t n_history,
                             const kreg_registration_config* config, double* next) {
  return guarded([&] { *next = anneal_step(lengthscale, history, n_history, *config); });
}

kreg_status kreg_line_search(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z, const double T[12],
                             const double g[6], const kreg_kernel_params* params, const kreg_pairs* pairs,
                             const kreg_registration_config* config, double* step) {
  return guarded([&] {
    require(ctx && X && Z && T && g && params && pairs && config && step, "NULL argument");
    check_pairs_match(pairs, X, Z);
    // registration.cpp:86-98
    const double gnorm = kreg_se3::twist_norm6(g);
    if (!(gnorm > 0.0)) throw Error(KREG_INVALID_ARGUMENT, "line_search: gradient norm must be > 0");
    const int K = config->max_backtracks + 1;
    std::vector<double> Ts(static_cast<size_t>(K + 1) * 12), out(static_cast<size_t>(K + 1) * 8, 0.0);
    std::memcpy(Ts.data(), T, sizeof(double) * 12);
    std::vector<double> eps(static_cast<size_t>(K));
    double e = config->step_init * params->lengthscale;
    const double s = 1.0 / gnorm;
    for (int k = 0; k < K; ++k) {
      double tw[6], E[12];
      for (int t = 0; t < 6; ++t) tw[t] = (g[t] * s) * e;
      if (!kreg_se3::exp(tw, E)) throw Error(KREG_INVALID_ARGUMENT, "exp: twist has non-finite components");
      kreg_se3::compose(E, T, Ts.data() + 12 * (k + 1));
      eps[static_cast<size_t>(k)] = e;
      e *= config->step_shrink;
    }
    if (pairs->P > 0) eval_many(ctx, const_cast<kreg_pairs*>(pairs), Ts.data(), K + 1, params->lengthscale, params->sigma, out.data());
    *step = 0.0;
    for (int k = 0; k < K; ++k)
      if (out[8 * (k + 1)] > out[0]) {
        *step = eps[static_cast<size_t>(k)];
        break;
      }
  });
}

static void make_jobs(const kreg_cloud* X, const kreg_cloud* Z, const double* initial, const kreg_kernel_params* params,
                      const kreg_registration_config* config, kreg_registration_result* result, RegJob& j) {
  require(X && Z && initial && params && config && result, "NULL argument");
  j.X = X;
  j.Z = Z;
  std::memcpy(j.initial, initial, sizeof(j.initial));
  j.params = to_params(params);
  j.cfg = *config;
  j.out = result;
}

kreg_status kreg_register_clouds(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z, const double initial[12],
                                 const kreg_kernel_params* params, const kreg_registration_config* config,
                                 kreg_registration_result* result) {
  return guarded([&] {
    require(ctx != nullptr, "NULL context");
    std::vector<RegJob> jobs(1);
    make_jobs(X, Z, initial, params, config, result, jobs[0]);
    register_many(ctx, jobs);
    if (jobs[0].status != KREG_OK) throw Error(jobs[0].status, jobs[0].error);
  });
}

kreg_status kreg_register_clouds_rows(kreg_ctx* ctx, const kreg_cloud* X, const kreg_cloud* Z_rows,
                                      int64_t n_z_total, const double initial[12], const kreg_kernel_params* params,
                                      const kreg_registration_config* config, kreg_registration_result* result) {
  return guarded([&] {
    require(ctx != nullptr, "NULL context");
    require(Z_rows != nullptr && n_z_total >= Z_rows->n, "n_z_total must cover this rank's rows");
    std::vector<RegJob> jobs(1);
    make_jobs(X, Z_rows, initial, params, config, result, jobs[0]);
    jobs[0].n_z_total = n_z_total;
    register_many(ctx, jobs, &ctx->collective);
    if (jobs[0].status != KREG_OK) throw Error(jobs[0].status, jobs[0].error);
  });
}

kreg_status kreg_ctx_set_collective(kreg_ctx* ctx, kreg_collective_fn fn, void* user) {
  return guarded([&] {
    require(ctx != nullptr, "NULL context");
    nccl_detach(ctx);
    ctx->collective.fn = fn;
    ctx->collective.user = user;
  });
}

kreg_status kreg_ctx_timer_mark(kreg_ctx* ctx, int32_t which) {
  return guarded([&] {
    require(ctx != nullptr && (which == 0 || which == 1), "timer_mark: NULL context or bad mark");
    KREG_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->timer[which]) KREG_CUDA(cudaEventCreate(&ctx->timer[which]));
    KREG_CUDA(cudaEventRecord(ctx->timer[which], ctx->stream));
  });
}

kreg_status kreg_ctx_timer_elapsed(kreg_ctx* ctx, double* ms) {
  return guarded([&] {
    require(ctx != nullptr && ms != nullptr && ctx->timer[0] && ctx->timer[1], "timer_elapsed: marks missing");
    KREG_CUDA(cudaEventSynchronize(ctx->timer[1]));
    float f = 0.0f;
    KREG_CUDA(cudaEventElapsedTime(&f, ctx->timer[0], ctx->timer[1]));
    *ms = static_cast<double>(f);
  });
}

kreg_status kreg_nccl_unique_id(uint8_t id[128]) {
  return guarded([&] {
    require(id != nullptr, "NULL argument");
    nccl_unique_id(id);
  });
}

kreg_status kreg_ctx_set_nccl(kreg_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t world,
                              int32_t deterministic) {
  return guarded([&] {
    require(ctx != nullptr, "NULL context");
    if (world <= 0) {
      nccl_detach(ctx);
      return;
    }
    require(id != nullptr, "NULL unique id");
    nccl_attach(ctx, id, rank, world, deterministic != 0);
  });
}

int64_t kreg_ctx_nccl_calls(const kreg_ctx* ctx) { return ctx ? nccl_calls(ctx) : 0; }

kreg_status kreg_register_clouds_host(kreg_ctx* ctx, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                                      const double initial[12], const kreg_kernel_params* params,
                                      const kreg_registration_config* config, kreg_registration_result* result) {
  return guarded([&] {
    require(ctx && X && Z, "NULL argument");
    // staged on a worker thread into the context's upload arena (no device
    // allocation per call once the arena holds a pair of this size)
    const kreg_cloud_view* views[2] = {X, Z};
    std::unique_ptr<AsyncUpload> up = cloud_upload_async(ctx, views, 1);
    std::vector<RegJob> jobs(1);
    make_jobs(up->clouds[0].get(), up->clouds[1].get(), initial, params, config, result, jobs[0]);
    jobs[0].ready = &up->ready[0];
    jobs[0].ready_ev = up->done[0];
    try {
      register_many(ctx, jobs);
    } catch (...) {
      up.reset();  // join the worker before the clouds go away
      throw;
    }
    up.reset();
    if (jobs[0].status != KREG_OK) throw Error(jobs[0].status, jobs[0].error);
  });
}

kreg_status kreg_register_batch(kreg_ctx* ctx, int32_t n, const kreg_cloud* const* X, const kreg_cloud* const* Z,
                                const double* initials, const kreg_kernel_params* params,
                                const kreg_registration_config* config, kreg_registration_result* results,
                                int32_t* statuses) {
  return guarded([&] {
    require(ctx && (n == 0 || (X && Z && initials && results && statuses)), "NULL argument");
    std::vector<RegJob> jobs(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) make_jobs(X[k], Z[k], initials + 12 * k, params, config, &results[k], jobs[k]);
    register_many(ctx, jobs);
    for (int k = 0; k < n; ++k) statuses[k] = jobs[k].status;
  });
}

kreg_status kreg_register_batch_host(kreg_ctx* ctx, int32_t n, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                                     const double* initials, const kreg_kernel_params* params,
                                     const kreg_registration_config* config, kreg_registration_result* results,
                                     int32_t* statuses) {
  return guarded([&] {
    require(ctx && (n == 0 || (X && Z && initials && results && statuses)), "NULL argument");
    std::vector<const kreg_cloud_view*> views;
    for (int k = 0; k < n; ++k) {
      views.push_back(&X[k]);
      views.push_back(&Z[k]);
    }
    // clouds are staged and uploaded on worker threads while earlier
    // registrations already run (job k starts once its copies are enqueued)
    std::unique_ptr<AsyncUpload> up = cloud_upload_async(ctx, views.data(), n);
    std::vector<RegJob> jobs(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
      make_jobs(up->clouds[2 * k].get(), up->clouds[2 * k + 1].get(), initials + 12 * k, params, config, &results[k],
                jobs[k]);
      jobs[k].ready = &up->ready[static_cast<size_t>(k)];
      jobs[k].ready_ev = up->done[static_cast<size_t>(k)];
    }
    try {
      register_many(ctx, jobs);
    } catch (...) {
      up.reset();  // join the workers before the clouds go away
      throw;
    }
    up.reset();
    for (int k = 0; k < n; ++k) statuses[k] = jobs[k].status;
  });
}

kreg_status kreg_register_sequence(kreg_ctx* ctx, const kreg_cloud* const* frames, int32_t n_frames,
                                   const kreg_kernel_params* params, const kreg_registration_config* config,
                                   kreg_sequence_result* result) {
  return guarded([&] {
    // registration.cpp:191-230
    if (n_frames < 2) throw Error(KREG_INVALID_ARGUMENT, "register_sequence: need at least 2 frames");
    require(ctx && frames && params && config && result, "NULL argument");
    run_chains(ctx, frames, n_frames, {0}, {n_frames - 1}, to_params(params), *config, result);
  });
}

kreg_status kreg_register_sequence_chains(kreg_ctx* ctx, const kreg_cloud* const* frames, int32_t n_frames,
                                          int32_t n_chains, const kreg_kernel_params* params,
                                          const kreg_registration_config* config, kreg_sequence_result* result) {
  return guarded([&] {
    if (n_frames < 2) throw Error(KREG_INVALID_ARGUMENT, "register_sequence: need at least 2 frames");
    require(ctx && frames && params && config && result && n_chains >= 1, "invalid argument");
    const int m = n_frames - 1;
    const int nc = std::min(n_chains, m);
    std::vector<int> b, e;
    for (int c = 0; c < nc; ++c) {
      b.push_back(static_cast<int>(static_cast<long long>(m) * c / nc));
      e.push_back(static_cast<int>(static_cast<long long>(m) * (c + 1) / nc));
    }
    run_chains(ctx, frames, n_frames, b, e, to_params(params), *config, result);
  });
}

kreg_status kreg_register_sequence_host(kreg_ctx* ctx, const kreg_cloud_view* frames, int32_t n_frames,
                                        int32_t n_chains, const kreg_kernel_params* params,
                                        const kreg_registration_config* config, kreg_sequence_result* result) {
  return guarded([&] {
    if (n_frames < 2) throw Error(KREG_INVALID_ARGUMENT, "register_sequence: need at least 2 frames");
    require(ctx && frames && params && config && result && n_chains >= 1, "invalid argument");
    std::vector<const kreg_cloud_view*> views;
    for (int k = 0; k < n_frames; ++k) views.push_back(&frames[k]);
    const int m = n_frames - 1;
    const int nc = std::min(n_chains, m);
    std::vector<int> b, e;
    for (int c = 0; c < nc; ++c) {
      b.push_back(static_cast<int>(static_cast<long long>(m) * c / nc));
      e.push_back(static_cast<int>(static_cast<long long>(m) * (c + 1) / nc));
    }
    // frames are staged and uploaded on worker threads while the first pairs
    // already run, interleaved across the chains (frame k of every chain,
    // then k + 1, ...) so that every chain can start at once
    std::vector<int> order;
    std::vector<char> seen(static_cast<size_t>(n_frames), 0);
    for (int k = 0;; ++k) {
      bool any = false;
      for (int c = 0; c < nc; ++c) {
        const int f = b[c] + k;
        if (f > e[c]) continue;  // chain c covers frames b_c .. e_c
        any = true;
        if (!seen[static_cast<size_t>(f)]) {
          seen[static_cast<size_t>(f)] = 1;
          order.push_back(f);
        }
      }
      if (!any) break;
    }
    for (int f = 0; f < n_frames; ++f)
      if (!seen[static_cast<size_t>(f)]) order.push_back(f);
    std::unique_ptr<AsyncUpload> up = cloud_upload_async(ctx, views.data(), n_frames, 1, std::move(order));
    std::vector<const kreg_cloud*> fr;
    for (auto& c : up->clouds) fr.push_back(c.get());
    try {
      run_chains(ctx, fr.data(), n_frames, b, e, to_params(params), *config, result, up->ready.data(),
                 up->done.data());
    } catch (...) {
      up.reset();  // join the workers before the clouds go away
      throw;
    }
    up.reset();
  });
}

kreg_status kreg_register_sequence_spans(kreg_ctx* ctx, const kreg_cloud* const* frames, int32_t n_frames,
                                         const int32_t* begins, const int32_t* ends, int32_t n_spans,
                                         const kreg_kernel_params* params, const kreg_registration_config* config,
                                         kreg_sequence_result* result) {
  return guarded([&] {
    if (n_frames < 2) throw Error(KREG_INVALID_ARGUMENT, "register_sequence: need at least 2 frames");
    require(ctx && frames && params && config && result && begins && ends && n_spans >= 1, "invalid argument");
    std::vector<int> b, e;
    for (int s = 0; s < n_spans; ++s) {
      require(begins[s] >= 0 && begins[s] < ends[s] && ends[s] <= n_frames - 1, "span out of range");
      if (s) require(begins[s] >= ends[s - 1], "spans must be ordered and disjoint");
      b.push_back(begins[s]);
      e.push_back(ends[s]);
    }
    run_chains(ctx, frames, n_frames, b, e, to_params(params), *config, result);
  });
}

kreg_status kreg_indicator_sweep(kreg_ctx* ctx, const kreg_cloud_view* cloud, const kreg_kernel_params* params,
                                int32_t axis, double range, int32_t steps, double cutoff_multiplier, double c_min,
                                double* magnitudes, double* indicators) {
  return guarded([&] {
    // eval.cpp:198-235: indicator(cloud, perturb(cloud), I) at `steps`
    // magnitudes; indicator(X, P Z, I) == indicator(X, Z, P) (same FP64
    // apply), so every magnitude is one pair build + one evaluation at P,
    // all issued in one batched device round
    require(ctx && cloud && params && magnitudes && indicators, "NULL argument");
    require(axis == KREG_SWEEP_ROTATION || axis == KREG_SWEEP_TRANSLATION, "indicator_sweep: unknown axis");
    if (steps < 2 && range != 0.0) throw Error(KREG_INVALID_ARGUMENT, "indicator_sweep: steps must be >= 2");
    if (range < 0.0) throw Error(KREG_INVALID_ARGUMENT, "indicator_sweep: range must be >= 0");
    double centroid[3] = {0, 0, 0};
    for (int i = 0; i < cloud->n; ++i)
      for (int k = 0; k < 3; ++k) centroid[k] += cloud->xyz[3 * i + k];
    if (cloud->n > 0)
      for (double& v : centroid) v /= cloud->n;
    std::vector<double> mags;
    if (range == 0.0) {
      mags.push_back(0.0);
    } else {
      for (int k = 0; k < steps; ++k) mags.push_back(range * static_cast<double>(k) / static_cast<double>(steps - 1));
    }
    std::unique_ptr<kreg_cloud> c(cloud_create(ctx, cloud));
    const Params p = to_params(params);
    check_build_args(c.get(), c.get(), p, cutoff_multiplier, c_min);
    if (c->n == 0) throw Error(KREG_INVALID_ARGUMENT, "indicator: clouds must be non-empty");
    const size_t K = mags.size();
    std::vector<std::unique_ptr<kreg_pairs>> lists(K);
    std::vector<double> Ts(12 * K), outs(8 * K, 0.0);
    std::vector<BuildJob> builds;
    std::vector<EvalJob> evals;
    for (size_t k = 0; k < K; ++k) {
      double* T = Ts.data() + 12 * k;
      if (axis == KREG_SWEEP_ROTATION) {
        const double xi[6] = {0, 0, mags[k], 0, 0, 0};
        kreg_se3::exp(xi, T);  // rotation about z through the centroid
        for (int r = 0; r < 3; ++r)
          T[4 * r + 3] = centroid[r] - (T[4 * r] * centroid[0] + T[4 * r + 1] * centroid[1] + T[4 * r + 2] * centroid[2]);
      } else {
        kreg_se3::identity(T);
        T[3] = mags[k];
      }
      lists[k] = std::make_unique<kreg_pairs>();
      BuildJob b;
      b.pairs = lists[k].get();
      b.X = c.get();
      b.Z = c.get();
      std::memcpy(b.T, T, sizeof(b.T));
      b.params = p;
      b.cutoff_multiplier = cutoff_multiplier;
      b.c_min = c_min;
      builds.push_back(b);
      EvalJob e;
      e.pairs = lists[k].get();
      e.M = 1;
      std::memcpy(e.T[0], T, sizeof(double) * 12);
      e.lengthscale = p.lengthscale;
      e.sigma = p.sigma;
      e.out = outs.data() + 8 * k;
      evals.push_back(e);
    }
    run_round(ctx, builds, evals);
    const double denom = static_cast<double>(c->n);  // sqrt(|X| |Z|) with X == Z
    for (size_t k = 0; k < K; ++k) {
      magnitudes[k] = mags[k];
      indicators[k] = lists[k]->P > 0 ? outs[8 * k] / denom : 0.0;
    }
  });
}

// ---------------------------------------------------------------- ingest
}  // extern "C"
namespace {

void check_selector(const kreg_selector_config* sel) {  // selector.cpp:8-19
  require(sel != nullptr, "NULL argument");
  if (!(sel->target_min > 0 && sel->target_min < sel->target_max))
    throw Error(KREG_INVALID_ARGUMENT, "selector: need 0 < target_min < target_max");
  if (!(sel->initial_threshold > 0.0)) throw Error(KREG_INVALID_ARGUMENT, "selector: initial_threshold must be > 0");
  if (!(sel->adjust_factor > 1.0)) throw Error(KREG_INVALID_ARGUMENT, "selector: adjust_factor must be > 1");
}

void check_intr(const kreg_camera_intrinsics* in) {  // projection.cpp:7-20
  require(in != nullptr, "NULL argument");
  if (!(in->fx > 0.0 && in->fy > 0.0)) throw Error(KREG_INVALID_ARGUMENT, "intrinsics: fx and fy must be > 0");
  if (!(in->max_depth > 0.0)) throw Error(KREG_INVALID_ARGUMENT, "intrinsics: max_depth must be > 0");
  if (!(in->depth_scale > 0.0)) throw Error(KREG_INVALID_ARGUMENT, "intrinsics: depth_scale must be > 0");
  if (in->skip_top_rows < 0) throw Error(KREG_INVALID_ARGUMENT, "intrinsics: skip_top_rows must be >= 0");
}

// One frame: score + histogram on the device, the reference's threshold
// rounds on the host (selector.cpp:81-124) from the histogram, then the
// ordered compaction / back-projection when the caller's capacity suffices.
void run_ingest(kreg_ctx* ctx, const uint16_t* depth, const uint8_t* rgb, int channels, const float* sem, int sem_ch,
                const uint8_t* valid_mask, int w, int h, const kreg_camera_intrinsics* intr,
                const kreg_selector_config* sel, int32_t* pixels, double* xyz, double* feat, int64_t cap,
                kreg_selection_info* info) {
  require(rgb && info && w >= 0 && h >= 0 && (channels == 1 || channels >= 3) && sem_ch >= 0,
          "invalid ingest arguments");
  KREG_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t npx = static_cast<size_t>(w) * h;
  kreg_dev::IngestReq R{};
  R.w = w; R.h = h; R.channels = channels; R.sem_channels = sem ? sem_ch : 0;
  ctx->ing_rgb.ensure(npx * channels + 1);
  ctx->ing_score.ensure(npx + 1);
  ctx->ing_valid.ensure(npx + 1);
  ctx->ing_hist.ensure(256);
  if (npx) KREG_CUDA(cudaMemcpyAsync(ctx->ing_rgb.ptr, rgb, npx * channels, cudaMemcpyHostToDevice, st));
  R.rgb = ctx->ing_rgb.ptr;
  if (valid_mask) {
    ctx->ing_valid_in.ensure(npx + 1);
    if (npx) KREG_CUDA(cudaMemcpyAsync(ctx->ing_valid_in.ptr, valid_mask, npx, cudaMemcpyHostToDevice, st));
    R.valid_in = ctx->ing_valid_in.ptr;
  } else {
    ctx->ing_depth.ensure(npx + 1);
    if (npx) KREG_CUDA(cudaMemcpyAsync(ctx->ing_depth.ptr, depth, npx * sizeof(uint16_t), cudaMemcpyHostToDevice, st));
    R.depth = ctx->ing_depth.ptr;
    R.skip_top_rows = intr->skip_top_rows;
    R.depth_scale = intr->depth_scale; R.max_depth = intr->max_depth;
    R.fx = intr->fx; R.fy = intr->fy; R.cx = intr->cx; R.cy = intr->cy;
    if (sem && sem_ch > 0) {
      ctx->ing_sem.ensure(npx * sem_ch + 1);
      if (npx) KREG_CUDA(cudaMemcpyAsync(ctx->ing_sem.ptr, sem, npx * sem_ch * sizeof(float), cudaMemcpyHostToDevice, st));
      R.sem = ctx->ing_sem.ptr;
    }
  }
  R.score = ctx->ing_score.ptr;
  R.valid = ctx->ing_valid.ptr;
  R.hist = ctx->ing_hist.ptr;
  KREG_CUDA(cudaMemsetAsync(R.hist, 0, 256 * sizeof(unsigned long long), st));
  unsigned long long hist[256] = {};
  if (npx) {
    kreg_dev::ingest_score(R, st);
    KREG_CUDA(cudaMemcpyAsync(hist, R.hist, sizeof(hist), cudaMemcpyDeviceToHost, st));
    KREG_CUDA(cudaStreamSynchronize(st));
  }
  long long total_valid = 0;
  for (unsigned long long v : hist) total_valid += static_cast<long long>(v);
  // corner count at threshold t: valid interior pixels with score > t (the
  // reference's strict segment test at t; scores <= 0 never pass t >= 0.5)
  auto count = [&](double t) {
    long long c = 0;
    for (int s = 1; s < 256; ++s)
      if (static_cast<double>(s) > t) c += static_cast<long long>(hist[s]);
    return c;
  };
  constexpr double kMinThreshold = 0.5;  // selector.cpp:81
  double t = sel->initial_threshold, best_t = 0.0;
  long best_gap = -1;
  long long best_count = 0;
  bool in_band = false;
  for (int round = 0; round < sel->max_adjust_rounds; ++round) {
    const long long cnt = count(t);
    const long gap = cnt < sel->target_min ? sel->target_min - cnt : cnt > sel->target_max ? cnt - sel->target_max : 0;
    if (best_gap < 0 || gap < best_gap) {
      best_gap = gap;
      best_t = t;
      best_count = cnt;
    }
    if (gap == 0) {
      in_band = true;
      break;
    }
    if (cnt > sel->target_max) {
      t *= sel->adjust_factor;
    } else {
      if (t <= kMinThreshold) break;
      t = std::max(t / sel->adjust_factor, kMinThreshold);
    }
  }
  const bool fallback = !in_band && best_count < sel->target_min;
  info->count = fallback ? total_valid : best_count;
  info->threshold = best_t;
  info->in_band = in_band ? 1 : 0;
  info->fallback = fallback ? 1 : 0;
  info->valid_pixels = total_valid;
  const long long n = info->count;
  if (n == 0 || cap < n || !pixels) return;
  R.threshold = best_t;
  R.fallback = fallback ? 1 : 0;
  const int nb = kreg_dev::ingest_blocks(static_cast<long long>(npx));
  ctx->ing_block_count.ensure(nb + 1);
  ctx->ing_block_off.ensure(nb + 2);
  ctx->ing_pixels.ensure(2 * static_cast<size_t>(n));
  R.block_count = ctx->ing_block_count.ptr;
  R.block_off = ctx->ing_block_off.ptr;
  R.pixels = ctx->ing_pixels.ptr;
  R.cap = n;
  const int D = 3 + R.sem_channels;
  if (xyz && feat && !valid_mask) {
    ctx->ing_xyz.ensure(3 * static_cast<size_t>(n));
    ctx->ing_feat.ensure(static_cast<size_t>(D) * n);
    R.xyz = ctx->ing_xyz.ptr;
    R.feat = ctx->ing_feat.ptr;
  }
  kreg_dev::ingest_emit(R, true, st);
  kreg_dev::ingest_emit(R, false, st);
  KREG_CUDA(cudaMemcpyAsync(pixels, R.pixels, 2 * sizeof(int) * n, cudaMemcpyDeviceToHost, st));
  if (R.xyz) {
    KREG_CUDA(cudaMemcpyAsync(xyz, R.xyz, 3 * sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    KREG_CUDA(cudaMemcpyAsync(feat, R.feat, sizeof(double) * D * n, cudaMemcpyDeviceToHost, st));
  }
  KREG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace
extern "C" {

kreg_status kreg_select_points(kreg_ctx* ctx, const uint8_t* rgb, int32_t channels, int32_t width, int32_t height,
                               const uint8_t* valid_depth, const kreg_selector_config* sel, int32_t* pixels_uv,
                               int64_t capacity, kreg_selection_info* info) {
  return guarded([&] {
    require(ctx && valid_depth, "NULL argument");
    check_selector(sel);
    run_ingest(ctx, nullptr, rgb, channels, nullptr, 0, valid_depth, width, height, nullptr, sel, pixels_uv, nullptr,
               nullptr, capacity, info);
  });
}

kreg_status kreg_depth_rgb_to_cloud(kreg_ctx* ctx, const uint16_t* depth, const uint8_t* rgb, int32_t channels,
                                    const float* semantics, int32_t semantic_channels, int32_t width, int32_t height,
                                    const kreg_camera_intrinsics* intr, const kreg_selector_config* sel, double* xyz,
                                    double* features, int64_t capacity, kreg_selection_info* info) {
  return guarded([&] {
    require(ctx && depth, "NULL argument");
    check_intr(intr);
    check_selector(sel);
    // the pixel list is device scratch here; positions and features are the output
    std::vector<int32_t> px(capacity > 0 ? static_cast<size_t>(2 * capacity) : 0);
    run_ingest(ctx, depth, rgb, channels, semantics, semantic_channels, nullptr, width, height, intr, sel,
               px.empty() ? nullptr : px.data(), xyz, features, capacity, info);
  });
}

kreg_status kreg_exact_cosine(kreg_ctx* ctx, const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                              const kreg_kernel_params* params, double* cosine, double parts[3]) {
  return guarded([&] {
    // inner_product.cpp:203-236
    require(ctx && X && Z && T && params && cosine, "NULL argument");
    std::unique_ptr<kreg_cloud> cx(cloud_describe(ctx, X)), cz(cloud_describe(ctx, Z));
    check_same_schema(cx.get(), cz.get(), "");
    const Params p = to_params(params);
    check_kernel_params(p, cx.get());
    if (X->n == 0 || Z->n == 0) throw Error(KREG_INVALID_ARGUMENT, "exact_cosine: clouds must be non-empty");
    const int D = X->dim;
    if (D > kreg_dev::kMaxDenseDim)
      throw Error(KREG_INVALID_ARGUMENT, "exact_cosine: feature rows longer than 32 are not supported");
    KREG_CUDA(cudaSetDevice(ctx->device));
    // Z transformed on the host in FP64 exactly as apply(T, p) (se3.cpp:129-131)
    std::vector<double> tz(static_cast<size_t>(Z->n) * 3);
    for (int j = 0; j < Z->n; ++j) {
      const double* q = Z->xyz + 3 * j;
      for (int r = 0; r < 3; ++r)
        tz[3 * j + r] = T[4 * r] * q[0] + T[4 * r + 1] * q[1] + T[4 * r + 2] * q[2] + T[4 * r + 3];
    }
    const size_t nx = static_cast<size_t>(X->n), nz = static_cast<size_t>(Z->n);
    kreg_host::DevBuf<double> dx, dz, dtz, dfx, dfz, part;
    kreg_host::DevBuf<kreg_dev::DenseReq> dreq;
    dx.ensure(3 * nx, false, 1.0);
    dz.ensure(3 * nz, false, 1.0);
    dtz.ensure(3 * nz, false, 1.0);
    dfx.ensure(nx * D + 1, false, 1.0);
    dfz.ensure(nz * D + 1, false, 1.0);
    KREG_CUDA(cudaMemcpyAsync(dx.ptr, X->xyz, sizeof(double) * 3 * nx, cudaMemcpyHostToDevice, ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(dz.ptr, Z->xyz, sizeof(double) * 3 * nz, cudaMemcpyHostToDevice, ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(dtz.ptr, tz.data(), sizeof(double) * 3 * nz, cudaMemcpyHostToDevice, ctx->stream));
    if (D) {
      KREG_CUDA(cudaMemcpyAsync(dfx.ptr, X->features, sizeof(double) * nx * D, cudaMemcpyHostToDevice, ctx->stream));
      KREG_CUDA(cudaMemcpyAsync(dfz.ptr, Z->features, sizeof(double) * nz * D, cudaMemcpyHostToDevice, ctx->stream));
    }
    const int b_chunks = 8;
    const int nb_a = kreg_dev::dense_blocks_a(static_cast<int>(std::max(nx, nz)));
    const size_t per = static_cast<size_t>(nb_a) * b_chunks;
    part.ensure(3 * per, false, 1.0);
    kreg_dev::DenseReq h[3];
    std::memset(h, 0, sizeof(h));
    const double* apos[3] = {dx.ptr, dx.ptr, dz.ptr};
    const double* bpos[3] = {dtz.ptr, dx.ptr, dz.ptr};
    const double* afe[3] = {dfx.ptr, dfx.ptr, dfz.ptr};
    const double* bfe[3] = {dfz.ptr, dfx.ptr, dfz.ptr};
    const int na[3] = {X->n, X->n, Z->n}, nb[3] = {Z->n, X->n, Z->n};
    double pref = p.sigma * p.sigma;
    int off = 0;
    for (size_t k = 0; k < p.per_channel.size(); ++k) {
      const kreg_channel_params& cp = p.per_channel[k];
      if (cp.form != KREG_FORM_LINEAR) pref *= cp.sigma * cp.sigma;
    }
    for (int r = 0; r < 3; ++r) {
      h[r].a = apos[r];
      h[r].b = bpos[r];
      h[r].af = afe[r];
      h[r].bf = bfe[r];
      h[r].n_a = na[r];
      h[r].n_b = nb[r];
      h[r].D = D;
      h[r].n_channels = static_cast<int>(p.per_channel.size());
      off = 0;
      for (int k = 0; k < h[r].n_channels; ++k) {
        const kreg_channel_params& cp = p.per_channel[static_cast<size_t>(k)];
        h[r].ch[k].offset = off;
        h[r].ch[k].dim = cx->schema[static_cast<size_t>(k)].dim;
        h[r].ch[k].linear = cp.form == KREG_FORM_LINEAR ? 1 : 0;
        h[r].ch[k].neg_inv_2l2 = cp.form == KREG_FORM_LINEAR ? 0.0 : -1.0 / (2.0 * cp.lengthscale * cp.lengthscale);
        off += h[r].ch[k].dim;
      }
      h[r].neg_inv_2l2 = -1.0 / (2.0 * p.lengthscale * p.lengthscale);
      h[r].pref = pref;
      h[r].partials = part.ptr + r * per;
    }
    dreq.ensure(3, false, 1.0);
    KREG_CUDA(cudaMemcpyAsync(dreq.ptr, h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
    kreg_dev::dense_sums(h, dreq.ptr, 3, b_chunks, ctx->stream);
    KREG_CUDA(cudaGetLastError());
    std::vector<double> hp(3 * per);
    KREG_CUDA(cudaMemcpyAsync(hp.data(), part.ptr, sizeof(double) * 3 * per, cudaMemcpyDeviceToHost, ctx->stream));
    KREG_CUDA(cudaStreamSynchronize(ctx->stream));
    double s[3];
    for (int r = 0; r < 3; ++r) {
      double t = 0.0;
      for (size_t k = 0; k < per; ++k) t += hp[r * per + k];  // fixed order
      s[r] = t;
    }
    if (!(s[1] > 0.0) || !(s[2] > 0.0)) throw Error(KREG_INVALID_ARGUMENT, "exact_cosine: zero-norm cloud function");
    *cosine = s[0] / std::sqrt(s[1] * s[2]);
    if (parts) {
      parts[0] = s[0];
      parts[1] = s[1];
      parts[2] = s[2];
    }
  });
}

kreg_status kreg_se3_exp(const double xi[6], double out[12]) {
  return guarded([&] {
    if (!kreg_se3::exp(xi, out)) throw Error(KREG_INVALID_ARGUMENT, "exp: twist has non-finite components");
  });
}

void kreg_se3_compose(const double a[12], const double b[12], double out[12]) { kreg_se3::compose(a, b, out); }
void kreg_se3_inverse(const double T[12], double out[12]) { kreg_se3::inverse(T, out); }
double kreg_cloud_diameter(const kreg_cloud_view* view) { return diameter_host(view->xyz, view->n); }

}  // extern "C"

