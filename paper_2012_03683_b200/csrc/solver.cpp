// Host registration loop (reference registration.cpp:100-189), written as a
// per-registration state machine so that any number of independent
// registrations advance in lockstep on one device: every round issues the
// batched pair builds and candidate sweeps of all active registrations, then
// one D2H + synchronize, then each state machine consumes its results.
//
// Parity contract: identical decisions to the
// reference given identical F/grad values — rebuild rule, skip rule, step
// candidates eps_k = step0 * shrink^k (running product), first F > f0
// accepted, step_factor adaptation, traces, convergence and annealing. The
// device differs only in HOW it evaluates:
//  * the line-search candidates are evaluated K at a time (with gradient and
//    displacement), and the accepted candidate's gradient is reused as the
//    next iteration's objective_and_gradient at the same T and pair list
//    (bitwise what a fresh evaluation would return: the sweep is
//    deterministic and independent of batch composition);
//  * candidate values are memoised across iterations while (T, dir, pair
//    list) are unchanged (a failed search re-tries the same candidates with
//    a halved step, registration.cpp:154).
#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <thread>
#include <vector>

#include "engine_host.hpp"
#include "se3_host.hpp"
#include "solver.hpp"

namespace kreg_host {

double anneal_step(double lengthscale, const double* hist, int n, const kreg_registration_config& c) {
  // registration.cpp:36-52
  const int window = c.stabilization_window;
  if (n < window) return lengthscale;
  const double* last = hist + (n - window);
  double lo = last[0], hi = last[0], scale = std::abs(last[0]);
  for (int k = 0; k < window; ++k) {
    lo = std::min(lo, last[k]);
    hi = std::max(hi, last[k]);
    scale = std::max(scale, std::abs(last[k]));
  }
  if (hi - lo > c.stabilization_rel_tol * std::max(scale, DBL_MIN)) return lengthscale;
  const double decayed = lengthscale * c.decay_factor;
  return decayed >= c.min_lengthscale ? decayed : lengthscale;
}

kreg_pairs* acquire_workspace(kreg_ctx* ctx) {
  kreg_pairs* p = nullptr;
  if (ctx && !ctx->pool.empty()) {
    p = ctx->pool.back();
    ctx->pool.pop_back();
  } else {
    p = new kreg_pairs;
  }
  p->ctx = ctx;
  p->X = p->Z = nullptr;
  p->built_at_lengthscale = 0.0;
  p->cutoff_radius = 0.0;
  p->P = 0;
  p->sup_valid = false;
  return p;
}

void release_workspace(kreg_ctx* ctx, kreg_pairs* p) {
  if (ctx && ctx->pool.size() < 512) {
    ctx->pool.push_back(p);
  } else {
    delete p;
  }
}

namespace {
template <class T>
long long held(const DevBuf<T>& b) {
  return b.ptr && b.owned ? static_cast<long long>(b.cap * sizeof(T)) : 0;
}
}  // namespace

long long workspace_bytes(const kreg_pairs* p) {
  return held(p->sup) + held(p->sup_i) + held(p->sup_count) + held(p->sup_off) + held(p->count) + held(p->perm) +
         held(p->pos) + held(p->deg_s) + held(p->tile_off) + held(p->slot_buf) + held(p->slot_i) +
         held(p->unit_off) + held(p->zs) + held(p->chunks) + held(p->disp_blk) + held(p->alt_perm) +
         held(p->alt_pos) + held(p->alt_deg_s) + held(p->alt_unit_off) + held(p->alt_tile_off) +
         held(p->alt_slot_buf) + held(p->alt_zs) + held(p->alt_chunks);
}

long long workspace_estimate(const kreg_ctx* ctx) {
  // candidate entries + indices, sweep slots + indices (+ the refilter's
  // second slot buffer), plus the per-source arrays
  const long long slot_bytes = static_cast<long long>(sizeof(int4) + sizeof(int)) * ctx->hw_slots;
  return static_cast<long long>(sizeof(int4) + sizeof(int)) * ctx->hw_sup + slot_bytes +
         (ctx->refilter ? slot_bytes : 0) + (16LL << 20);
}

namespace {

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

struct Memo {
  double eps;
  bool grad;  // out[1..6] holds the gradient
  double out[kreg_dev::kOut];
};

// Pair-list workspace borrowed from the context pool for one registration.
struct WsHandle {
  kreg_ctx* ctx = nullptr;
  kreg_pairs* p = nullptr;
  WsHandle() = default;
  WsHandle(const WsHandle&) = delete;
  WsHandle& operator=(const WsHandle&) = delete;
  ~WsHandle() { reset(); }
  kreg_pairs* get() const { return p; }
  kreg_pairs* operator->() const { return p; }
  void reset() {
    if (p) release_workspace(ctx, p);
    p = nullptr;
  }
};

enum class Phase { kInit, kStartIter, kAwaitEval, kSearchSetup, kSearch, kAwaitCandidates, kDone };

struct Reg {
  RegJob* job = nullptr;
  kreg_registration_config cfg{};
  Params wp;
  WsHandle pairs;
  double v_scale = 1.0, denom = 1.0;
  double lengthscale = 0.0;
  double T[12];
  std::vector<double> window;
  double step_factor = 1.0;
  // evaluation at T with the current pair list
  bool have_eval = false;
  double ev[kreg_dev::kOut];  // F, omega, v, disp
  bool rebuilt = false;       // this iteration rebuilt the pair list
  bool awaiting_build = false;
  // line search
  double dir[6];
  double step0 = 0.0;
  int k_next = 0;            // next candidate index
  double eps_next = 0.0;     // eps of candidate k_next
  std::vector<Memo> memo;    // candidates known for (T, dir, pairs)
  int pending = 0;           // candidates in flight
  double cand_T[24][12];
  double cand_eps[24];
  double cand_out[24][kreg_dev::kOut];
  bool cand_grad = true;     // the in-flight candidates carry their gradient
  // outputs
  std::vector<double> tr_obj, tr_ind, tr_l, tr_step, tr_tn;
  std::vector<long long> tr_pc;
  std::vector<uint8_t> tr_rb;
  bool converged = false;
  Phase phase = Phase::kInit;
  int sweeps = 0, rebuilds = 0;
};

void finish(Reg& r) {
  RegJob& j = *r.job;
  kreg_registration_result* o = j.out;
  std::memcpy(o->transform, r.T, sizeof(r.T));
  o->converged = r.converged ? 1 : 0;
  o->iterations = static_cast<int>(r.tr_obj.size());
  o->final_indicator = r.tr_ind.empty() ? 0.0 : r.tr_ind.back();
  const int n = std::min(o->trace_capacity, o->iterations);
  for (int i = 0; i < n; ++i) {
    if (o->objective_trace) o->objective_trace[i] = r.tr_obj[i];
    if (o->indicator_trace) o->indicator_trace[i] = r.tr_ind[i];
    if (o->lengthscale_trace) o->lengthscale_trace[i] = r.tr_l[i];
    if (o->step_trace) o->step_trace[i] = r.tr_step[i];
    if (o->twist_norm_trace) o->twist_norm_trace[i] = r.tr_tn[i];
    if (o->pair_count_trace) o->pair_count_trace[i] = r.tr_pc[i];
    if (o->rebuild_trace) o->rebuild_trace[i] = r.tr_rb[i];
  }
  o->sweeps = r.sweeps;
  o->rebuilds = r.rebuilds;
  j.status = KREG_OK;
  r.phase = Phase::kDone;
  r.pairs.reset();
}

// Optional line-search statistics (KREG_STATS=1): accepted backtrack index
// histogram (index 21 = search failed), printed to stderr at exit.
struct SearchStats {
  long long hist[22] = {};
  long long level_builds = 0, level_subset = 0;  // level-change rebuilds; of them, new pairs within the old list
  bool on = std::getenv("KREG_STATS") != nullptr;
  ~SearchStats() {
    if (!on) return;
    std::fprintf(stderr, "kreg level-change rebuilds %lld, of which moved < cutoff shrink: %lld\n", level_builds,
                 level_subset);
    std::fprintf(stderr, "kreg line-search accepted-k histogram:");
    for (int k = 0; k < 22; ++k) std::fprintf(stderr, " %lld", hist[k]);
    std::fprintf(stderr, "\n");
  }
};
SearchStats g_search_stats;

// End of one reference iteration (registration.cpp:145-182).
void end_iteration(Reg& r, bool searched, bool accepted, int backtracks, double eps, const double* cand_T,
                   const double* cand_out, bool cand_has_grad = true) {
  const kreg_registration_config& c = r.cfg;
  double accepted_step = 0.0, twist_norm = 0.0, f_now = r.ev[0];
  if (searched && g_search_stats.on) ++g_search_stats.hist[accepted ? std::min(backtracks, 20) : 21];
  if (searched) {
    if (accepted) {
      accepted_step = eps;
      f_now = cand_out[0];
      double applied[6];
      for (int k = 0; k < 6; ++k) applied[k] = r.dir[k] * accepted_step;
      std::memcpy(r.T, cand_T, sizeof(r.T));  // == compose(exp(applied), T)
      twist_norm = std::sqrt(applied[0] * applied[0] + applied[1] * applied[1] + applied[2] * applied[2]) +
                   std::sqrt(applied[3] * applied[3] + applied[4] * applied[4] + applied[5] * applied[5]) / r.v_scale;
      r.step_factor = backtracks == 0 ? std::min(r.step_factor * c.step_grow, 1e3)
                                      : std::max(r.step_factor * std::pow(c.step_shrink, backtracks), 1e-6);
      // F, grad and displacement at the new T (an F-only candidate leaves the
      // gradient to a fresh evaluation at the start of the next iteration)
      std::memcpy(r.ev, cand_out, sizeof(r.ev));
      r.have_eval = cand_has_grad;
      r.memo.clear();
    } else {
      r.step_factor = std::max(r.step_factor * c.step_shrink, 1e-6);
    }
  }
  const double ind = f_now / r.denom;
  r.tr_l.push_back(r.lengthscale);
  r.tr_obj.push_back(f_now);
  r.tr_ind.push_back(ind);
  r.tr_step.push_back(accepted_step);
  r.tr_tn.push_back(twist_norm);
  r.tr_pc.push_back(r.pairs->P);
  r.tr_rb.push_back(r.rebuilt ? 1 : 0);
  r.window.push_back(ind);

  const bool at_floor = r.lengthscale * c.decay_factor < c.min_lengthscale;
  if (at_floor && twist_norm < c.convergence_twist_norm) {
    r.converged = true;
    finish(r);
    return;
  }
  const double next = anneal_step(r.lengthscale, r.window.data(), static_cast<int>(r.window.size()), c);
  if (next != r.lengthscale) {
    r.lengthscale = next;
    r.wp.lengthscale = next;
    r.window.clear();
    r.step_factor = 1.0;
  }
  r.phase = Phase::kStartIter;
}

// The displacement max_j |T z_j - T_build z_j| the loop's decisions need
// (EvalJob::disp_limit): the rebuild rule compares it with 0.5 cutoff
// (registration.cpp:123-128), the next build's candidate-list reuse with
// R_s - 2 margin - sup_disp - cutoff_next (prepare_build), cutoff_next in
// {cutoff, decay x cutoff} (one anneal step at most). Any value at or below
// the returned limit leads to the same decisions as the exact maximum.
double disp_limit(const Reg& r) {
  const kreg_pairs* p = r.pairs.get();
  double lim = 0.5 * p->cutoff_radius;
  if (p->sup_valid) {
    const double base = p->sup_radius - 2e-9 * p->sup_radius - p->sup_disp;
    for (const double cut : {p->cutoff_radius, p->cutoff_radius * r.cfg.decay_factor}) {
      const double b = base - cut;
      if (b >= 0.0) lim = std::min(lim, b);
    }
  }
  return lim * (1.0 - 1e-12);
}

void schedule_build_eval(Reg& r, std::vector<BuildJob>& builds, std::vector<EvalJob>& evals,
                         std::vector<Reg*>& eval_owner) {
  BuildJob b;
  b.pairs = r.pairs.get();
  b.X = r.job->X;
  b.Z = r.job->Z;
  std::memcpy(b.T, r.T, sizeof(r.T));
  b.params = r.wp;
  b.cutoff_multiplier = r.cfg.cutoff_multiplier;
  b.c_min = r.cfg.c_min;
  // displacement of T from the current list's build transform (from the
  // sweep that evaluated T); lets the engine filter its candidate list
  b.disp_hint = r.phase == Phase::kInit ? -1.0 : r.ev[7];
  if (r.phase == Phase::kInit) {  // the first build reads the uploaded clouds
    b.wait_ev[0] = r.job->ready_ev;
    b.wait_ev[1] = r.job->ready_ev2;
  }
  builds.push_back(b);
  EvalJob e;
  e.pairs = r.pairs.get();
  e.M = 1;
  std::memcpy(e.T[0], r.T, sizeof(r.T));
  e.lengthscale = r.lengthscale;
  e.sigma = r.wp.sigma;
  e.out = r.ev;
  e.disp_limit = disp_limit(r);
  evals.push_back(e);
  eval_owner.push_back(&r);
  r.memo.clear();
  r.have_eval = false;
  r.awaiting_build = true;
  ++r.rebuilds;
  ++r.sweeps;
}

// Advance host-only logic until the registration needs device work.
void plan(Reg& r, std::vector<BuildJob>& builds, std::vector<EvalJob>& evals, std::vector<Reg*>& owners,
          int k_first, bool fail_grad) {
  const kreg_registration_config& c = r.cfg;
  for (;;) {
    switch (r.phase) {
      case Phase::kDone:
      case Phase::kAwaitEval:
      case Phase::kAwaitCandidates:
        return;
      case Phase::kInit:
        // registration.cpp:110-115: initial build at T0 (+ the first evaluation)
        schedule_build_eval(r, builds, evals, owners);
        r.phase = Phase::kAwaitEval;
        return;
      case Phase::kStartIter: {
        if (static_cast<int>(r.tr_obj.size()) >= c.max_iterations) {
          finish(r);
          return;
        }
        // registration.cpp:123-128 rebuild rule (displacement of T vs T_build
        // comes from the sweep that evaluated T)
        r.rebuilt = false;
        if (r.pairs->built_at_lengthscale != r.lengthscale || r.ev[7] > 0.5 * r.pairs->cutoff_radius ||
            !r.have_eval) {
          const bool must = r.pairs->built_at_lengthscale != r.lengthscale || r.ev[7] > 0.5 * r.pairs->cutoff_radius;
          if (must) {
            if (g_search_stats.on && r.pairs->built_at_lengthscale != r.lengthscale && r.have_eval) {
              ++g_search_stats.level_builds;
              if (r.ev[7] <= r.pairs->cutoff_radius - r.cfg.cutoff_multiplier * r.lengthscale)
                ++g_search_stats.level_subset;
            }
            r.rebuilt = true;
            schedule_build_eval(r, builds, evals, owners);
            r.phase = Phase::kAwaitEval;
            return;
          }
          EvalJob e;
          e.pairs = r.pairs.get();
          e.M = 1;
          std::memcpy(e.T[0], r.T, sizeof(r.T));
          e.lengthscale = r.lengthscale;
          e.sigma = r.wp.sigma;
          e.out = r.ev;
          e.disp_limit = disp_limit(r);
          evals.push_back(e);
          owners.push_back(&r);
          ++r.sweeps;
          r.phase = Phase::kAwaitEval;
          return;
        }
        r.phase = Phase::kSearchSetup;
        break;
      }
      case Phase::kSearchSetup: {
        const double* g = r.ev + 1;
        const double gnorm = kreg_se3::twist_norm6(g);
        r.step0 = c.step_init * r.lengthscale * r.step_factor;  // registration.cpp:132
        // registration.cpp:139 skip rule
        if (gnorm > 0.0 && r.step0 * gnorm > 1e-12 * std::max(std::abs(r.ev[0]), 1.0)) {
          const double s = 1.0 / gnorm;
          double dir[6];
          for (int k = 0; k < 6; ++k) dir[k] = g[k] * s;
          if (std::memcmp(dir, r.dir, sizeof(dir)) != 0) r.memo.clear();
          std::memcpy(r.dir, dir, sizeof(dir));
          r.k_next = 0;
          r.eps_next = r.step0;
          r.phase = Phase::kSearch;
        } else {
          end_iteration(r, false, false, 0, 0.0, nullptr, nullptr);
          if (r.phase == Phase::kDone) return;
        }
        break;
      }
      case Phase::kSearch: {
        // registration.cpp:63-75: candidates k = k_next.. with eps_k = step0 * shrink^k
        const int remaining = c.max_backtracks + 1 - r.k_next;
        const int K = std::min(remaining, r.k_next == 0 ? k_first : 24);
        // resolve memoised candidates first (same T, dir, pair list)
        int n_new = 0;
        r.pending = 0;
        double eps = r.eps_next;
        bool resolved = false;
        const int k0 = r.k_next;
        for (int m = 0; m < K; ++m) {
          const int k = k0 + m;
          const Memo* hit = nullptr;
          for (const Memo& mm : r.memo)
            if (mm.eps == eps) hit = &mm;
          double cand[12], tw[6], E[12];
          for (int t = 0; t < 6; ++t) tw[t] = r.dir[t] * eps;
          kreg_se3::exp(tw, E);
          kreg_se3::compose(E, r.T, cand);
          if (hit && n_new == 0) {
            if (hit->out[0] > r.ev[0]) {
              end_iteration(r, true, true, k, eps, cand, hit->out, hit->grad);
              resolved = true;
              break;
            }
            r.k_next = k + 1;
            r.eps_next = eps * c.step_shrink;
          } else {
            std::memcpy(r.cand_T[n_new], cand, sizeof(cand));
            r.cand_eps[n_new] = eps;
            ++n_new;
          }
          eps *= c.step_shrink;
        }
        if (resolved) {
          if (r.phase == Phase::kDone) return;
          break;
        }
        if (n_new == 0) {
          if (r.k_next > c.max_backtracks) {
            end_iteration(r, true, false, 0, 0.0, nullptr, nullptr);
            if (r.phase == Phase::kDone) return;
          }
          break;  // continue searching (more memo hits or new candidates)
        }
        // the first batch carries gradients (its accepted candidate's gradient
        // is the next iteration's); the failure-path batches evaluate F only
        r.cand_grad = k0 == 0 || fail_grad;
        for (int b = 0; b < n_new; b += kreg_dev::kMaxCandidates) {
          EvalJob e;
          e.pairs = r.pairs.get();
          e.M = std::min(kreg_dev::kMaxCandidates, n_new - b);
          for (int m = 0; m < e.M; ++m) std::memcpy(e.T[m], r.cand_T[b + m], sizeof(double) * 12);
          e.lengthscale = r.lengthscale;
          e.sigma = r.wp.sigma;
          e.out = &r.cand_out[b][0];
          e.disp_limit = disp_limit(r);
          e.grad = r.cand_grad;
          evals.push_back(e);
          owners.push_back(&r);
          ++r.sweeps;
        }
        r.pending = n_new;
        r.phase = Phase::kAwaitCandidates;
        return;
      }
    }
  }
}

void consume(Reg& r) {
  const kreg_registration_config& c = r.cfg;
  if (r.phase == Phase::kAwaitEval) {
    if (r.awaiting_build) {
      r.awaiting_build = false;
      if (r.pairs->P == 0) {
        if (r.tr_obj.empty() && !r.rebuilt) {
          // registration.cpp:115
          char msg[160];
          std::snprintf(msg, sizeof(msg), "no overlapping pairs within cutoff radius %f m", r.pairs->cutoff_radius);
          r.job->status = KREG_NO_OVERLAP;
          r.job->error = msg;
          r.phase = Phase::kDone;
          r.pairs.reset();
          return;
        }
        finish(r);  // registration.cpp:127: drifted out of support, unconverged
        return;
      }
    }
    r.have_eval = true;
    r.phase = Phase::kSearchSetup;
    return;
  }
  if (r.phase == Phase::kAwaitCandidates) {
    for (int m = 0; m < r.pending; ++m) {
      Memo mm;
      mm.eps = r.cand_eps[m];
      mm.grad = r.cand_grad;
      std::memcpy(mm.out, r.cand_out[m], sizeof(mm.out));
      r.memo.push_back(mm);
    }
    for (int m = 0; m < r.pending; ++m) {
      const int k = r.k_next + m;
      if (r.cand_out[m][0] > r.ev[0]) {
        double T[12], out[kreg_dev::kOut];
        std::memcpy(T, r.cand_T[m], sizeof(T));
        std::memcpy(out, r.cand_out[m], sizeof(out));
        end_iteration(r, true, true, k, r.cand_eps[m], T, out, r.cand_grad);
        return;
      }
    }
    r.k_next += r.pending;
    r.eps_next = r.cand_eps[r.pending - 1] * c.step_shrink;
    if (r.k_next > c.max_backtracks) {
      end_iteration(r, true, false, 0, 0.0, nullptr, nullptr);
    } else {
      r.phase = Phase::kSearch;
    }
  }
}

}  // namespace

// Combine a finished round across ranks: F, omega, v and pair counts are
// summed, displacements maxed (each rank holds disjoint source rows).
void reduce_round(RoundSlot& S, const Collective& coll) {
  std::vector<double> sums, maxes;
  for (const EvalJob& e : S.evals)
    for (int m = 0; m < e.M; ++m) {
      for (int k = 0; k < 7; ++k) sums.push_back(e.out[m * kreg_dev::kOut + k]);
      maxes.push_back(e.out[m * kreg_dev::kOut + 7]);
    }
  for (const BuildJob& b : S.builds) sums.push_back(static_cast<double>(b.pairs->P));
  if (coll.fn(coll.user, sums.data(), static_cast<int32_t>(sums.size()), maxes.data(),
              static_cast<int32_t>(maxes.size())) != 0)
    throw Error(KREG_CUDA_ERROR, "collective callback failed");
  size_t a = 0, b = 0;
  for (EvalJob& e : S.evals)
    for (int m = 0; m < e.M; ++m) {
      for (int k = 0; k < 7; ++k) e.out[m * kreg_dev::kOut + k] = sums[a++];
      e.out[m * kreg_dev::kOut + 7] = maxes[b++];
    }
  for (BuildJob& bj : S.builds) bj.pairs->P = static_cast<long long>(sums[a++]);
}

void register_many(kreg_ctx* ctx, std::vector<RegJob>& jobs, const Collective* coll) {
  NvtxScope nvtx("kreg.register_many");
  const int k_first = std::max(1, std::min(8, env_int("KREG_K_FIRST", 2)));
  const bool fail_grad = env_int("KREG_FAIL_GRAD", 0) != 0;
  std::vector<std::unique_ptr<Reg>> regs;
  std::vector<Reg*> job_reg(jobs.size(), nullptr);
  for (RegJob& j : jobs) {
    j.status = KREG_OK;
    auto r = std::make_unique<Reg>();
    r->job = &j;
    try {
      check_config(j.cfg);                          // registration.cpp:102
      check_same_schema(j.X, j.Z, "register: ");    // :103-104
      Params p0 = j.params;
      p0.lengthscale = j.cfg.init_lengthscale;
      check_kernel_params(p0, j.X);
      if (!(j.cfg.cutoff_multiplier >= 1.0))
        throw Error(KREG_INVALID_ARGUMENT, "build_pairs: cutoff_multiplier must be >= 1");
    } catch (const Error& e) {
      j.status = e.code;
      j.error = e.what();
      continue;
    }
    r->cfg = j.cfg;
    r->wp = j.params;
    const double diam = j.X->diam;
    r->v_scale = diam > 0.0 ? diam : 1.0;
    const long long nz = j.n_z_total > 0 ? j.n_z_total : j.Z->n;
    r->denom = std::sqrt(static_cast<double>(std::max(j.X->n, 1)) * static_cast<double>(std::max(nz, 1LL)));
    r->lengthscale = j.cfg.init_lengthscale;
    r->wp.lengthscale = r->lengthscale;
    std::memcpy(r->T, j.initial, sizeof(r->T));
    for (double& d : r->dir) d = 0.0;
    if (j.n_z_total > 0 && j.Z->n == 0) {
      j.status = KREG_INVALID_ARGUMENT;  // a rank without rows would leave the lockstep
      j.error = "register_clouds_rows: every rank needs at least one source row";
      continue;
    }
    if (j.X->n == 0 || j.Z->n == 0) {
      // empty cloud: build_pairs yields an empty list -> NoOverlapError
      char msg[160];
      std::snprintf(msg, sizeof(msg), "no overlapping pairs within cutoff radius %f m",
                    j.cfg.cutoff_multiplier * j.cfg.init_lengthscale);
      j.status = KREG_NO_OVERLAP;
      j.error = msg;
      continue;
    }
    job_reg[static_cast<size_t>(&j - jobs.data())] = r.get();
    regs.push_back(std::move(r));
  }
  // Ready queue: jobs without a predecessor in order; a chained job joins
  // when its predecessor finishes (resolve), with the initial guess
  // register_sequence gives it (registration.cpp:211-219).
  std::deque<Reg*> ready;
  std::function<void(int)> resolve = [&](int i) {
    const int s = jobs[static_cast<size_t>(i)].succ;
    if (s < 0) return;
    RegJob& J = jobs[static_cast<size_t>(i)];
    RegJob& S = jobs[static_cast<size_t>(s)];
    std::memcpy(S.initial, J.status == KREG_OK ? J.out->transform : J.initial, sizeof(S.initial));
    if (Reg* rs = job_reg[static_cast<size_t>(s)]) {
      std::memcpy(rs->T, S.initial, sizeof(rs->T));
      ready.push_back(rs);
    } else {
      resolve(s);  // failed before it could start (empty cloud): falls back at once
    }
  };
  for (size_t i = 0; i < jobs.size(); ++i) {
    if (jobs[i].pred >= 0) continue;
    if (job_reg[i]) ready.push_back(job_reg[i]);
    else resolve(static_cast<int>(i));
  }

  using clk = std::chrono::steady_clock;
  // At most `window` registrations are in flight; a finished one is replaced
  // by the next job at once (dynamic refill), so one slow registration does
  // not hold the batch. The active registrations form two groups whose
  // rounds alternate on the device: while one group's round runs, the host
  // consumes and plans the other's (the stream orders the rounds). Results
  // do not depend on the window or the grouping: every sweep request is
  // evaluated independently of what else shares its launch.
  const size_t window = ctx && ctx->max_active > 0 ? static_cast<size_t>(ctx->max_active) : regs.size();
  constexpr int kMaxGroups = 4;
  const int n_groups =
      ctx ? std::max(1, static_cast<int>(std::min<size_t>(
                            window, static_cast<size_t>(std::clamp(env_int("KREG_GROUPS", 2), 1, kMaxGroups)))))
          : 1;
  size_t started = 0;
  struct Group {
    std::vector<Reg*> active;
    std::vector<Reg*> owners;
    RoundSlot* slot = nullptr;
    bool pending = false;  // a round of this group is in flight
  };
  Group groups[kMaxGroups];
  // two groups: each on its own stream (slots 3 and 1), so their rounds
  // overlap on the device; both order after the context stream's uploads
  // several groups: each on its own stream (round slots 3, 1, 4, 5), so
  // their rounds overlap on the device; all order after the context stream's
  // uploads. One group runs on the context stream (slot 0).
  for (int g = 0; g < n_groups; ++g) groups[g].slot = round_slot(ctx, n_groups == 1 ? 0 : (g == 0 ? 3 : g == 1 ? 1 : g + 2));
  const size_t per_group = (window + n_groups - 1) / n_groups;

  // Memory-aware admission: a registration starts only when the device has
  // room for its workspace at the context's high-water capacities (every
  // workspace grows to those). A registration whose first candidate radius
  // exceeds any radius built so far (the first call on a context, or the
  // first-frame schedule after subsequent pairs) starts alone and the rest
  // wait one round for its build to size the estimate. One registration is
  // always admitted when nothing is in flight.
  auto in_flight = [&] {
    size_t n = 0;
    for (int g = 0; g < n_groups; ++g) n += groups[g].active.size();
    return n;
  };
  // workspace bytes admitted in this refill pass but not allocated yet (the
  // builds that grow them run after the pass)
  long long admit_pending = 0;
  long long mem_free = -1;  // free device bytes minus a reserve, queried once per refill pass
  auto admit = [&](const Reg* r) -> bool {
    if (!ctx || in_flight() == 0) return true;
    const double rs = r->cfg.cutoff_multiplier * r->cfg.init_lengthscale * (1.0 + std::max(0.0, ctx->skin));
    if (rs > ctx->hw_radius * (1.0 + 1e-9)) return false;
    if (ctx->mem_budget > 0)
      return static_cast<long long>(in_flight() + 1) * workspace_estimate(ctx) <= ctx->mem_budget;
    long long need = workspace_estimate(ctx);
    if (!ctx->pool.empty()) need -= workspace_bytes(ctx->pool.back());
    if (need <= 0) return true;
    need += need / 4;
    if (mem_free < 0) {  // one query per refill pass (cudaMemGetInfo costs up to ~1 ms)
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return true;
      }
      mem_free = static_cast<long long>(free_b) - std::max<long long>(1LL << 30, static_cast<long long>(total_b / 50));
    }
    if (mem_free < admit_pending + need) return false;
    admit_pending += need;
    return true;
  };

  // host phase trace (KREG_TRACE_HOST=1): per-round microseconds of
  // end_round after the wait, consume, refill + plan, begin_round
  static const bool trace_host = std::getenv("KREG_TRACE_HOST") != nullptr;
  double ph[4] = {0, 0, 0, 0};
  long long ph_rounds = 0;
  const double wait0 = ctx ? ctx->t_wait : 0.0;
  auto us = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  // consume the finished round of group g, refill, plan and launch its next
  auto step = [&](Group& G) -> bool {
    const auto t0 = clk::now();
    if (G.pending) {
      end_round(ctx, *G.slot);
      if (coll && coll->fn) reduce_round(*G.slot, *coll);
      G.pending = false;
      const auto t1 = clk::now();
      if (trace_host) ph[0] += us(t0, t1);
      Reg* last = nullptr;
      for (Reg* r : G.owners) {  // each registration consumes once per round
        if (r == last) continue;
        last = r;
        consume(*r);
      }
      if (ctx) ctx->t_total += std::chrono::duration<double>(clk::now() - t1).count();
      if (trace_host) ph[1] += us(t1, clk::now());
    }
    const auto t2 = clk::now();
    for (;;) {
      for (Reg* r : G.active)  // finished chain links release their successors
        if (r->phase == Phase::kDone) resolve(static_cast<int>(r->job - jobs.data()));
      G.active.erase(std::remove_if(G.active.begin(), G.active.end(), [](Reg* r) { return r->phase == Phase::kDone; }),
                     G.active.end());
      admit_pending = 0;
      mem_free = -1;
      while (G.active.size() < per_group && !ready.empty()) {
        // end-to-end batches: start a job once its clouds' copies are enqueued
        const RegJob* fj = ready.front()->job;
        if (fj->ready || fj->ready2) {
          auto state = [fj] {
            const int a = fj->ready ? fj->ready->load(std::memory_order_acquire) : 1;
            const int b = fj->ready2 ? fj->ready2->load(std::memory_order_acquire) : 1;
            return a < 0 || b < 0 ? -1 : std::min(a, b);
          };
          int v = state();
          while (v == 0 && in_flight() == 0) {  // nothing else to run: wait for the upload
            std::this_thread::yield();
            v = state();
          }
          if (v < 0) throw Error(KREG_CUDA_ERROR, "cloud upload failed");
          if (v == 0) break;
        }
        if (!admit(ready.front())) {
          if (ctx) ++ctx->deferred_admissions;
          break;
        }
        Reg* r = ready.front();
        ready.pop_front();
        ++started;
        r->pairs.ctx = ctx;
        r->pairs.p = acquire_workspace(ctx);
        if (r->job->expected_pairs > 0) r->pairs->expected_pairs = r->job->expected_pairs;
        G.active.push_back(r);
        if (ctx) ctx->peak_in_flight = std::max<long long>(ctx->peak_in_flight, static_cast<long long>(in_flight()));
      }
      std::vector<BuildJob> builds;
      std::vector<EvalJob> evals;
      G.owners.clear();
      for (Reg* r : G.active) plan(*r, builds, evals, G.owners, k_first, fail_grad);
      if (!builds.empty() || !evals.empty()) {
        if (ctx) ctx->t_total += std::chrono::duration<double>(clk::now() - t2).count();
        const auto t3 = clk::now();
        begin_round(ctx, *G.slot, std::move(builds), std::move(evals));
        if (trace_host) {
          ph[2] += us(t2, t3);
          ph[3] += us(t3, clk::now());
          ++ph_rounds;
        }
        G.pending = true;
        (void)t0;
        return true;
      }
      if (ready.empty() && G.active.empty()) return false;  // group drained
      if (G.active.empty()) return true;  // waiting for memory: the other group runs
      // every active registration finished without device work: refill
    }
  };
  bool live[kMaxGroups];
  for (int g = 0; g < kMaxGroups; ++g) live[g] = g < n_groups;
  auto any_live = [&] {
    for (int g = 0; g < n_groups; ++g)
      if (live[g]) return true;
    return false;
  };
  while (any_live()) {
    for (int g = 0; g < n_groups; ++g)
      if (live[g]) live[g] = step(groups[g]);
  }
  if (trace_host && ph_rounds) {
    const double n = static_cast<double>(ph_rounds), wait = ctx ? (ctx->t_wait - wait0) * 1e6 : 0.0;
    std::fprintf(stderr,
                 "kreg-host rounds %lld  us/round: end_round %.1f (wait %.1f), consume %.1f, plan %.1f, begin_round %.1f\n",
                 ph_rounds, ph[0] / n, wait / n, ph[1] / n, ph[2] / n, ph[3] / n);
  }
}

}  // namespace kreg_host
