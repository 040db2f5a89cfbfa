// kreg_b200/kreg.hpp — C++ layer over the C-ABI in ../kreg_b200.h.
//
// Owns the ABI handles (RAII), turns status codes back into the exceptions
// the reference throws, and carries the reference's value types as plain
// arrays so that it needs no Eigen. The reference-typed API itself
// (kreg::build_pairs, kreg::register_clouds, ... with kreg::PointCloud /
// Isometry / PairList, /root/reference/proj/include/kreg/{inner_product,
// registration}.hpp) is implemented on top of this header by
// paper_2012_03683_b200/facade/kreg_facade.cpp, which a maintainer compiles
// into the reference build in place of inner_product.cpp and
// registration.cpp.
//
// Exception mapping (reference errors.hpp:9-36):
//   KREG_INVALID_ARGUMENT -> std::invalid_argument
//   KREG_NO_OVERLAP       -> kreg_b200::NoOverlapError (cutoff_radius())
//   KREG_PARSE_ERROR      -> kreg_b200::ParseError
//   KREG_OUT_OF_MEMORY    -> std::bad_alloc
//   everything else       -> std::runtime_error
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../kreg_b200.h"

namespace kreg_b200 {

class NoOverlapError : public std::runtime_error {
 public:
  NoOverlapError(const std::string& what, double cutoff_radius)
      : std::runtime_error(what), cutoff_radius_(cutoff_radius) {}
  double cutoff_radius() const { return cutoff_radius_; }

 private:
  double cutoff_radius_;
};

class ParseError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// The cutoff radius named in a no-overlap message ("... cutoff radius R m").
inline double cutoff_from_message(const std::string& m) {
  const auto at = m.find("radius ");
  return at == std::string::npos ? 0.0 : std::strtod(m.c_str() + at + 7, nullptr);
}

[[noreturn]] inline void throw_status(kreg_status s, const std::string& what) {
  switch (s) {
    case KREG_INVALID_ARGUMENT:
      throw std::invalid_argument(what);
    case KREG_NO_OVERLAP:
      throw NoOverlapError(what, cutoff_from_message(what));
    case KREG_PARSE_ERROR:
      throw ParseError(what);
    case KREG_OUT_OF_MEMORY:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(what);
  }
}

inline void check(kreg_status s) {
  if (s != KREG_OK) throw_status(s, kreg_last_error());
}

// --------------------------------------------------------------- handles
struct CtxFree {
  void operator()(kreg_ctx* c) const { kreg_ctx_destroy(c); }
};
struct CloudFree {
  void operator()(kreg_cloud* c) const { kreg_cloud_destroy(c); }
};
struct PairsFree {
  void operator()(kreg_pairs* p) const { kreg_pairs_destroy(p); }
};

// One CUDA device + stream (not thread-safe: serialise calls per context).
class Context {
 public:
  explicit Context(int device = 0) {
    kreg_ctx* c = nullptr;
    check(kreg_ctx_create(device, &c));
    h_.reset(c);
  }
  kreg_ctx* get() const { return h_.get(); }

 private:
  std::unique_ptr<kreg_ctx, CtxFree> h_;
};

// Kernel parameters with owned per-channel storage (kernels.hpp:16-33).
struct Params {
  double sigma = 1.0, lengthscale = 1.0;
  std::vector<kreg_channel_params> per_channel;
  kreg_kernel_params view() const {
    return kreg_kernel_params{sigma, lengthscale, per_channel.empty() ? nullptr : per_channel.data(),
                              static_cast<int32_t>(per_channel.size())};
  }
};

// Host view of a cloud with owned channel-name storage (point_cloud.hpp:17-76).
struct CloudView {
  const double* xyz = nullptr;  // n x 3
  int32_t n = 0;
  const double* features = nullptr;  // n x dim
  int32_t dim = 0;
  std::vector<std::string> names;
  std::vector<kreg_channel> channels;
  void add_channel(const std::string& name, int32_t d, int32_t kind) {
    names.push_back(name);
    channels.push_back(kreg_channel{nullptr, d, kind});
  }
  kreg_cloud_view view() const {
    std::vector<kreg_channel>& ch = const_cast<std::vector<kreg_channel>&>(channels);
    for (size_t k = 0; k < ch.size(); ++k) ch[k].name = names[k].c_str();
    return kreg_cloud_view{xyz, n, features, dim, ch.empty() ? nullptr : ch.data(), static_cast<int32_t>(ch.size())};
  }
};

// Device-resident cloud (uploaded once, immutable like the reference's).
class Cloud {
 public:
  Cloud() = default;
  Cloud(Context& ctx, const CloudView& v) {
    const kreg_cloud_view cv = v.view();
    kreg_cloud* c = nullptr;
    check(kreg_cloud_create(ctx.get(), &cv, &c));
    h_.reset(c);
    n_ = v.n;
  }
  const kreg_cloud* get() const { return h_.get(); }
  int size() const { return n_; }

 private:
  std::unique_ptr<kreg_cloud, CloudFree> h_;
  int n_ = 0;
};

// Reference PairList layout (inner_product.hpp:18-32).
struct Csr {
  std::vector<int64_t> offsets;
  std::vector<int32_t> x_index;
  std::vector<double> coeff;
};

// Device pair list (build_pairs, inner_product.cpp:37-95).
class Pairs {
 public:
  Pairs() = default;
  Pairs(Context& ctx, const Cloud& X, const Cloud& Z, const double T[12], const Params& p, double cutoff_multiplier,
        double c_min) {
    const kreg_kernel_params kp = p.view();
    kreg_pairs* h = nullptr;
    int64_t n = 0;
    check(kreg_build_pairs(ctx.get(), X.get(), Z.get(), T, &kp, cutoff_multiplier, c_min, &h, &n));
    h_.reset(h);
    n_z_ = Z.size();
  }
  kreg_pairs* get() const { return h_.get(); }
  int64_t size() const { return h_ ? kreg_pairs_size(h_.get()) : 0; }
  Csr export_csr(Context& ctx) const {
    Csr out;
    out.offsets.assign(static_cast<size_t>(n_z_) + 1, 0);
    out.x_index.resize(static_cast<size_t>(size()));
    out.coeff.resize(static_cast<size_t>(size()));
    check(kreg_pairs_export(ctx.get(), h_.get(), out.offsets.data(), out.x_index.data(), out.coeff.data()));
    return out;
  }

 private:
  std::unique_ptr<kreg_pairs, PairsFree> h_;
  int n_z_ = 0;
};

inline kreg_registration_config default_config() {
  kreg_registration_config c;
  kreg_registration_config_default(&c);
  return c;
}

// RegistrationResult (registration.hpp:45-60) with owned traces.
struct Registration {
  double transform[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
  bool converged = false;
  int iterations = 0;
  double final_indicator = 0.0;
  std::vector<double> objective, indicator, lengthscale, step, twist_norm;
  std::vector<int64_t> pair_count;
  std::vector<uint8_t> rebuild;
};

inline Registration register_clouds(Context& ctx, const Cloud& X, const Cloud& Z, const double initial[12],
                                    const Params& p, const kreg_registration_config& cfg) {
  Registration r;
  const size_t cap = static_cast<size_t>(cfg.max_iterations > 0 ? cfg.max_iterations : 0);
  r.objective.resize(cap);
  r.indicator.resize(cap);
  r.lengthscale.resize(cap);
  r.step.resize(cap);
  r.twist_norm.resize(cap);
  r.pair_count.resize(cap);
  r.rebuild.resize(cap);
  kreg_registration_result res;
  std::memset(&res, 0, sizeof(res));
  res.trace_capacity = static_cast<int32_t>(cap);
  res.objective_trace = r.objective.data();
  res.indicator_trace = r.indicator.data();
  res.lengthscale_trace = r.lengthscale.data();
  res.step_trace = r.step.data();
  res.twist_norm_trace = r.twist_norm.data();
  res.pair_count_trace = r.pair_count.data();
  res.rebuild_trace = r.rebuild.data();
  const kreg_kernel_params kp = p.view();
  check(kreg_register_clouds(ctx.get(), X.get(), Z.get(), initial, &kp, &cfg, &res));
  std::memcpy(r.transform, res.transform, sizeof(r.transform));
  r.converged = res.converged != 0;
  r.iterations = res.iterations;
  r.final_indicator = res.final_indicator;
  const size_t n = static_cast<size_t>(res.iterations) < cap ? static_cast<size_t>(res.iterations) : cap;
  for (auto* v : {&r.objective, &r.indicator, &r.lengthscale, &r.step, &r.twist_norm}) v->resize(n);
  r.pair_count.resize(n);
  r.rebuild.resize(n);
  return r;
}

// SequenceResult (registration.hpp:85-92).
struct Sequence {
  std::vector<double> relative;    // (frames - 1) x 12
  std::vector<double> trajectory;  // frames x 12
  std::vector<uint8_t> fallback, converged;
  std::vector<double> final_indicator;
  std::vector<int32_t> iterations;
};

inline Sequence register_sequence(Context& ctx, const std::vector<const kreg_cloud*>& frames, const Params& p,
                                  const kreg_registration_config& cfg) {
  const size_t n = frames.size(), m = n > 0 ? n - 1 : 0;
  Sequence s;
  s.relative.resize(12 * m);
  s.trajectory.resize(12 * n);
  s.fallback.resize(m);
  s.converged.resize(m);
  s.final_indicator.resize(m);
  s.iterations.resize(m);
  kreg_sequence_result r{s.relative.data(), s.trajectory.data(), s.fallback.data(), s.converged.data(),
                         s.final_indicator.data(), s.iterations.data()};
  const kreg_kernel_params kp = p.view();
  check(kreg_register_sequence(ctx.get(), frames.data(), static_cast<int32_t>(n), &kp, &cfg, &r));
  return s;
}

}  // namespace kreg_b200
