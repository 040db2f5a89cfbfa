// TEST INFRASTRUCTURE: links the product's host solver (csrc/solver.cpp) to a
// CPU stand-in for the device round executor built on the C oracle, so the
// solver's state machine (rebuild rule, K-candidate batching, gradient reuse,
// memoisation, traces, annealing) can be checked against the reference's
// registration loop on a machine without a GPU. Never part of the product.
#include <cstring>
#include <map>
#include <vector>

#include "../../oracle/kreg_oracle.h"
#include "../../paper_2012_03683_b200/csrc/engine_host.hpp"
#include "../../paper_2012_03683_b200/csrc/solver.hpp"

namespace {
std::map<const kreg_cloud*, const kreg_cloud_view*> g_views;
std::map<const kreg_pairs*, ko_pairs*> g_pairs;
}  // namespace

namespace kreg_host {
void throw_cuda(cudaError_t, const char* what) { throw Error(KREG_CUDA_ERROR, what); }
void set_last_error(const std::string&) {}
const char* last_error() { return ""; }
void check_config(const kreg_registration_config& c) {
  if (ko_check_config(&c)) throw Error(KREG_INVALID_ARGUMENT, ko_last_error());
}
void check_same_schema(const kreg_cloud*, const kreg_cloud*, const char*) {}
void check_kernel_params(const Params&, const kreg_cloud*) {}

static kreg_kernel_params to_c(const Params& p, double l) {
  kreg_kernel_params k;
  k.sigma = p.sigma;
  k.lengthscale = l;
  k.per_channel = p.per_channel.data();
  k.n_channels = static_cast<int>(p.per_channel.size());
  return k;
}

void run_round(kreg_ctx*, std::vector<BuildJob>& builds, std::vector<EvalJob>& evals) {
  for (BuildJob& b : builds) {
    kreg_pairs* p = b.pairs;
    if (g_pairs.count(p)) ko_pairs_destroy(g_pairs[p]);
    const kreg_kernel_params kp = to_c(b.params, b.params.lengthscale);
    ko_pairs* op = nullptr;
    int64_t n = 0;
    ko_build_pairs(g_views[b.X], g_views[b.Z], b.T, &kp, b.cutoff_multiplier, b.c_min, 0, &op, &n);
    g_pairs[p] = op;
    p->X = b.X;
    p->Z = b.Z;
    p->P = n;
    p->built_at_lengthscale = b.params.lengthscale;
    p->cutoff_radius = b.cutoff_multiplier * b.params.lengthscale;
    p->sigma = b.params.sigma;
    std::memcpy(p->T_build, b.T, sizeof(p->T_build));
  }
  for (EvalJob& e : evals) {
    kreg_pairs* p = e.pairs;
    Params dummy;
    dummy.sigma = p->sigma;
    // per-channel params are irrelevant for the sweep (c is cached)
    const kreg_kernel_params kp = to_c(dummy, e.lengthscale);
    for (int m = 0; m < e.M; ++m) {
      double o[7];
      ko_objective_and_gradient(g_pairs[p], g_views[p->X], g_views[p->Z], e.T[m], &kp, o);
      std::memcpy(e.out + 8 * m, o, sizeof(o));
      e.out[8 * m + 7] = ko_max_point_displacement(g_views[p->Z], p->T_build, e.T[m]);
    }
  }
}

// the oracle evaluates synchronously: begin_round does the work, end_round
// has nothing to wait for
RoundSlot::~RoundSlot() {}
RoundSlot* round_slot(kreg_ctx*, int i) {
  static RoundSlot slots[3];
  return &slots[i];
}
void begin_round(kreg_ctx* ctx, RoundSlot& S, std::vector<BuildJob>&& builds, std::vector<EvalJob>&& evals) {
  S.builds = std::move(builds);
  S.evals = std::move(evals);
  run_round(ctx, S.builds, S.evals);
  S.in_flight = true;
}
void end_round(kreg_ctx*, RoundSlot& S) { S.in_flight = false; }
}  // namespace kreg_host

// registers once through the product solver with the oracle standing in for the device
extern "C" int mock_register_rows(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double initial[12],
                                  const kreg_kernel_params* params, const kreg_registration_config* config,
                                  kreg_registration_result* result, int k_first, long long n_z_total,
                                  kreg_collective_fn fn, void* user);

extern "C" int mock_register(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double initial[12],
                             const kreg_kernel_params* params, const kreg_registration_config* config,
                             kreg_registration_result* result, int k_first) {
  return mock_register_rows(X, Z, initial, params, config, result, k_first, 0, nullptr, nullptr);
}

// registers this rank's source rows Z through the product solver (oracle as
// the device); per-round results are combined through `fn` (row sharding)
extern "C" int mock_register_rows(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double initial[12],
                                  const kreg_kernel_params* params, const kreg_registration_config* config,
                                  kreg_registration_result* result, int k_first, long long n_z_total,
                                  kreg_collective_fn fn, void* user) {
  kreg_cloud cx, cz;
  cx.n = X->n;
  cz.n = Z->n;
  cx.diam = ko_diameter(X);
  g_views[&cx] = X;
  g_views[&cz] = Z;
  std::vector<kreg_host::RegJob> jobs(1);
  kreg_host::RegJob& j = jobs[0];
  j.X = &cx;
  j.Z = &cz;
  std::memcpy(j.initial, initial, sizeof(j.initial));
  j.params.sigma = params->sigma;
  j.params.lengthscale = params->lengthscale;
  for (int k = 0; k < params->n_channels; ++k) j.params.per_channel.push_back(params->per_channel[k]);
  j.cfg = *config;
  j.out = result;
  j.n_z_total = n_z_total;
  setenv("KREG_K_FIRST", std::to_string(k_first).c_str(), 1);
  kreg_host::Collective coll;
  coll.fn = fn;
  coll.user = user;
  kreg_host::register_many(nullptr, jobs, fn ? &coll : nullptr);
  for (auto& kv : g_pairs) ko_pairs_destroy(kv.second);
  g_pairs.clear();
  g_views.clear();
  return j.status;
}
