// Drop-in implementation of the reference's registration hot path on the
// B200 engine: the 13 functions that /root/reference/proj/src/inner_product.cpp
// and registration.cpp define, with the reference's own declarations
// (include/kreg/inner_product.hpp:50-87, include/kreg/registration.hpp:42-100),
// value types (PointCloud, Isometry, Twist, PairList, RegistrationResult,
// SequenceResult) and exceptions (std::invalid_argument, kreg::NoOverlapError).
//
// Build: compile this file inside the reference build in place of
// inner_product.cpp and registration.cpp, with the reference's include
// directory, this repository's include/ and its Eigen; link
// paper_2012_03683_b200/libkreg_b200.so. The reference's own
// unit tests test_inner_product.cpp / test_registration.cpp link against it
// unmodified (oracle/Makefile facade-tests, tests/test_facade.py).
//
// Every computation runs on the device through the C-ABI; there is no CPU
// path (an unavailable device raises std::runtime_error). Device state:
//  * one context per process (device KREG_DEVICE, default 0), created on
//    first use;
//  * clouds are uploaded once and cached by content (positions, features,
//    schema; the reference's PointCloud is immutable, point_cloud.hpp:48-50);
//  * a PairList returned by build_pairs keeps its device list in a cache keyed
//    by its storage; a PairList the cache does not know (copied, or made
//    elsewhere) is rebuilt on the device from the build inputs it records
//    (build_transform, built_at_lengthscale, cutoff_radius, c_min), which
//    yields the same list (builds are deterministic).
#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <vector>

#include "kreg/errors.hpp"
#include "kreg/inner_product.hpp"
#include "kreg/registration.hpp"
#include "kreg_b200/kreg.hpp"

namespace kreg {
namespace {

static_assert(sizeof(Eigen::Vector3d) == 3 * sizeof(double), "positions must be packed xyz triples");

using kreg_b200::check;

void to12(const Isometry& T, double out[12]) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) out[4 * r + c] = T.rotation(r, c);
    out[4 * r + 3] = T.translation(r);
  }
}

Isometry from12(const double* a) {
  Isometry T;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) T.rotation(r, c) = a[4 * r + c];
    T.translation(r) = a[4 * r + 3];
  }
  return T;
}

kreg_b200::Params to_params(const KernelParams& p) {
  kreg_b200::Params out;
  out.sigma = p.sigma;
  out.lengthscale = p.lengthscale;
  for (const ChannelParams& c : p.per_channel)
    out.per_channel.push_back(kreg_channel_params{c.sigma, c.lengthscale, static_cast<int32_t>(c.form)});
  return out;
}

kreg_registration_config to_config(const RegistrationConfig& c) {
  kreg_registration_config o;
  o.init_lengthscale = c.init_lengthscale;
  o.subsequent_lengthscale = c.subsequent_lengthscale;
  o.min_lengthscale = c.min_lengthscale;
  o.decay_factor = c.decay_factor;
  o.stabilization_window = c.stabilization_window;
  o.stabilization_rel_tol = c.stabilization_rel_tol;
  o.max_iterations = c.max_iterations;
  o.step_init = c.step_init;
  o.step_shrink = c.step_shrink;
  o.step_grow = c.step_grow;
  o.max_backtracks = c.max_backtracks;
  o.convergence_twist_norm = c.convergence_twist_norm;
  o.cutoff_multiplier = c.cutoff_multiplier;
  o.c_min = c.c_min;
  return o;
}

kreg_b200::CloudView view_of(const PointCloud& c) {
  kreg_b200::CloudView v;
  v.xyz = c.empty() ? nullptr : reinterpret_cast<const double*>(c.positions().data());
  v.n = c.size();
  v.features = c.features().empty() ? nullptr : c.features().data();
  v.dim = c.feature_dim();
  for (const Channel& ch : c.schema().channels()) v.add_channel(ch.name, ch.dim, static_cast<int32_t>(ch.kind));
  return v;
}

// Engine exceptions -> the reference's.
template <typename F>
auto translate(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const kreg_b200::NoOverlapError& e) {
    throw NoOverlapError(e.cutoff_radius());
  } catch (const kreg_b200::ParseError& e) {
    throw std::runtime_error(e.what());
  }
}

uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  return h * 0xFF51AFD7ED558CCDull;
}

uint64_t fingerprint(const PointCloud& c) {
  uint64_t h = mix(0x6B72656762323030ull, static_cast<uint64_t>(c.size()));
  auto words = [&](const void* p, size_t bytes) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i + 8 <= bytes; i += 8) {
      uint64_t w;
      std::memcpy(&w, b + i, 8);
      h = mix(h, w);
    }
  };
  if (!c.empty()) words(c.positions().data(), sizeof(double) * 3 * static_cast<size_t>(c.size()));
  if (!c.features().empty()) words(c.features().data(), sizeof(double) * c.features().size());
  for (const Channel& ch : c.schema().channels()) {
    h = mix(h, static_cast<uint64_t>(ch.dim) * 8 + static_cast<uint64_t>(ch.kind));
    for (char x : ch.name) h = mix(h, static_cast<unsigned char>(x));
  }
  return h;
}

struct CloudEntry {
  uint64_t fp = 0;
  int n = 0;
  std::unique_ptr<kreg_b200::Cloud> cloud;
  uint64_t used = 0;
};

struct PairEntry {
  const int32_t* data = nullptr;
  int64_t size = 0;
  const kreg_b200::Cloud* X = nullptr;
  const kreg_b200::Cloud* Z = nullptr;
  double T[12] = {};
  double lengthscale = 0.0, cutoff = 0.0, c_min = 0.0;
  std::unique_ptr<kreg_b200::Pairs> pairs;
  uint64_t used = 0;
};

constexpr size_t kMaxClouds = 32;
constexpr size_t kMaxPairs = 32;

struct Engine {
  std::mutex mu;  // the reference API is callable from any thread; one device context serialises it
  std::unique_ptr<kreg_b200::Context> ctx;
  std::vector<CloudEntry> clouds;
  std::vector<PairEntry> pairs;
  uint64_t clock = 0;

  kreg_b200::Context& context() {
    if (!ctx) {
      const char* d = std::getenv("KREG_DEVICE");
      ctx = std::make_unique<kreg_b200::Context>(d ? std::atoi(d) : 0);
    }
    return *ctx;
  }

  const kreg_b200::Cloud& cloud(const PointCloud& c) {
    const uint64_t fp = fingerprint(c);
    for (CloudEntry& e : clouds) {
      if (e.fp == fp && e.n == c.size()) {
        e.used = ++clock;
        return *e.cloud;
      }
    }
    if (clouds.size() >= kMaxClouds) {
      auto lru = std::min_element(clouds.begin(), clouds.end(),
                                  [](const CloudEntry& a, const CloudEntry& b) { return a.used < b.used; });
      const kreg_b200::Cloud* gone = lru->cloud.get();
      std::erase_if(pairs, [&](const PairEntry& p) { return p.X == gone || p.Z == gone; });
      clouds.erase(lru);
    }
    CloudEntry e;
    e.fp = fp;
    e.n = c.size();
    e.cloud = std::make_unique<kreg_b200::Cloud>(context(), view_of(c));
    e.used = ++clock;
    clouds.push_back(std::move(e));
    return *clouds.back().cloud;
  }

  void remember(const PairList& pl, const kreg_b200::Cloud& X, const kreg_b200::Cloud& Z,
                std::unique_ptr<kreg_b200::Pairs> dev) {
    if (pairs.size() >= kMaxPairs) {
      pairs.erase(std::min_element(pairs.begin(), pairs.end(),
                                   [](const PairEntry& a, const PairEntry& b) { return a.used < b.used; }));
    }
    PairEntry e;
    e.data = pl.x_index.data();
    e.size = pl.size();
    e.X = &X;
    e.Z = &Z;
    to12(pl.build_transform, e.T);
    e.lengthscale = pl.built_at_lengthscale;
    e.cutoff = pl.cutoff_radius;
    e.c_min = pl.c_min;
    e.pairs = std::move(dev);
    e.used = ++clock;
    pairs.push_back(std::move(e));
  }

  // the device list of a PairList (cached, else rebuilt from its build inputs)
  const kreg_b200::Pairs& device_pairs(const PairList& pl, const PointCloud& Xh, const PointCloud& Zh,
                                       const KernelParams& params) {
    const kreg_b200::Cloud& X = cloud(Xh);
    const kreg_b200::Cloud& Z = cloud(Zh);
    double T[12];
    to12(pl.build_transform, T);
    for (PairEntry& e : pairs) {
      if (e.data == pl.x_index.data() && e.size == pl.size() && e.X == &X && e.Z == &Z &&
          e.lengthscale == pl.built_at_lengthscale && e.cutoff == pl.cutoff_radius && e.c_min == pl.c_min &&
          std::memcmp(e.T, T, sizeof(T)) == 0) {
        e.used = ++clock;
        return *e.pairs;
      }
    }
    if (pl.n_x != Xh.size() || pl.n_z != Zh.size())
      throw std::invalid_argument("pair list was built for clouds of a different size");
    kreg_b200::Params p = to_params(params);
    p.lengthscale = pl.built_at_lengthscale;
    const double mult = pl.built_at_lengthscale > 0.0 ? pl.cutoff_radius / pl.built_at_lengthscale : 1.0;
    auto dev = std::make_unique<kreg_b200::Pairs>(context(), X, Z, T, p, std::max(1.0, mult), pl.c_min);
    if (dev->size() != pl.size())
      throw std::runtime_error("pair list does not match a device build from its recorded inputs");
    remember(pl, X, Z, std::move(dev));
    return *pairs.back().pairs;
  }
};

Engine& engine() {
  static Engine e;
  return e;
}

}  // namespace

// ------------------------------------------------ inner_product.hpp:50-87
PairList build_pairs(const PointCloud& X, const PointCloud& Z, const Isometry& T, const KernelParams& params,
                     double cutoff_multiplier, double c_min) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    const kreg_b200::Cloud& Xd = E.cloud(X);
    const kreg_b200::Cloud& Zd = E.cloud(Z);
    double t[12];
    to12(T, t);
    auto dev = std::make_unique<kreg_b200::Pairs>(E.context(), Xd, Zd, t, to_params(params), cutoff_multiplier, c_min);
    kreg_b200::Csr csr = dev->export_csr(E.context());
    PairList out;
    out.offsets = std::move(csr.offsets);
    out.x_index = std::move(csr.x_index);
    out.coeff = std::move(csr.coeff);
    out.built_at_lengthscale = params.lengthscale;
    out.cutoff_radius = cutoff_multiplier * params.lengthscale;
    out.c_min = c_min;
    out.build_transform = T;
    out.n_x = X.size();
    out.n_z = Z.size();
    E.remember(out, Xd, Zd, std::move(dev));  // the vectors' storage moves with the returned list
    return out;
  });
}

double inner_product(const PairList& pairs, const PointCloud& X, const PointCloud& Z, const Isometry& T,
                     const KernelParams& params) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    const kreg_b200::Pairs& P = E.device_pairs(pairs, X, Z, params);
    double t[12], v = 0.0;
    to12(T, t);
    const kreg_b200::Params p = to_params(params);
    const kreg_kernel_params kp = p.view();
    check(kreg_inner_product(E.context().get(), P.get(), E.cloud(X).get(), E.cloud(Z).get(), t, &kp, &v));
    return v;
  });
}

Evaluation objective_and_gradient(const PairList& pairs, const PointCloud& X, const PointCloud& Z,
                                  const Isometry& T, const KernelParams& params) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    const kreg_b200::Pairs& P = E.device_pairs(pairs, X, Z, params);
    double t[12], o[7];
    to12(T, t);
    const kreg_b200::Params p = to_params(params);
    const kreg_kernel_params kp = p.view();
    check(kreg_objective_and_gradient(E.context().get(), P.get(), E.cloud(X).get(), E.cloud(Z).get(), t, &kp, o));
    Evaluation ev;
    ev.value = o[0];
    ev.grad.omega = Eigen::Vector3d(o[1], o[2], o[3]);
    ev.grad.v = Eigen::Vector3d(o[4], o[5], o[6]);
    return ev;
  });
}

Twist gradient(const PairList& pairs, const PointCloud& X, const PointCloud& Z, const Isometry& T,
               const KernelParams& params) {
  return objective_and_gradient(pairs, X, Z, T, params).grad;
}

AlignmentReport evaluate_alignment(const PairList& pairs, const PointCloud& X, const PointCloud& Z,
                                   const Isometry& T, const KernelParams& params) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    const kreg_b200::Pairs& P = E.device_pairs(pairs, X, Z, params);
    double t[12];
    to12(T, t);
    const kreg_b200::Params p = to_params(params);
    const kreg_kernel_params kp = p.view();
    AlignmentReport r;
    int64_t n = 0;
    check(kreg_evaluate_alignment(E.context().get(), P.get(), E.cloud(X).get(), E.cloud(Z).get(), t, &kp,
                                  &r.value_F, &r.indicator, &n));
    r.pair_count = n;
    return r;
  });
}

double indicator(const PointCloud& X, const PointCloud& Z, const Isometry& T, const KernelParams& params,
                 double cutoff_multiplier, double c_min) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    double t[12], v = 0.0;
    to12(T, t);
    const kreg_b200::Params p = to_params(params);
    const kreg_kernel_params kp = p.view();
    check(kreg_indicator(E.context().get(), E.cloud(X).get(), E.cloud(Z).get(), t, &kp, cutoff_multiplier, c_min,
                         &v));
    return v;
  });
}

double exact_cosine(const PointCloud& X, const PointCloud& Z, const Isometry& T, const KernelParams& params) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    double t[12], v = 0.0;
    to12(T, t);
    const kreg_b200::Params p = to_params(params);
    const kreg_kernel_params kp = p.view();
    const kreg_b200::CloudView xv = view_of(X), zv = view_of(Z);
    const kreg_cloud_view xc = xv.view(), zc = zv.view();
    check(kreg_exact_cosine(E.context().get(), &xc, &zc, t, &kp, &v, nullptr));
    return v;
  });
}

double max_point_displacement(const PointCloud& Z, const Isometry& built, const Isometry& now) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    double a[12], b[12], v = 0.0;
    to12(built, a);
    to12(now, b);
    check(kreg_max_point_displacement(E.context().get(), E.cloud(Z).get(), a, b, &v));
    return v;
  });
}

// ------------------------------------------------ registration.hpp:42-100
void check_config(const RegistrationConfig& config) {
  const kreg_registration_config c = to_config(config);
  check(kreg_check_config(&c));
}

double anneal_step(double lengthscale, std::span<const double> indicator_history, const RegistrationConfig& config) {
  const kreg_registration_config c = to_config(config);
  double next = lengthscale;
  check(kreg_anneal_step(lengthscale, indicator_history.data(), static_cast<int32_t>(indicator_history.size()), &c,
                         &next));
  return next;
}

double line_search(const PointCloud& X, const PointCloud& Z, const Isometry& T, const Twist& g,
                   const KernelParams& params, const PairList& pairs, const RegistrationConfig& config) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    const kreg_b200::Pairs& P = E.device_pairs(pairs, X, Z, params);
    double t[12], step = 0.0;
    to12(T, t);
    const double gg[6] = {g.omega.x(), g.omega.y(), g.omega.z(), g.v.x(), g.v.y(), g.v.z()};
    const kreg_b200::Params p = to_params(params);
    const kreg_kernel_params kp = p.view();
    const kreg_registration_config c = to_config(config);
    check(kreg_line_search(E.context().get(), E.cloud(X).get(), E.cloud(Z).get(), t, gg, &kp, P.get(), &c, &step));
    return step;
  });
}

RegistrationResult register_clouds(const PointCloud& X, const PointCloud& Z, const Isometry& initial,
                                   const KernelParams& params, const RegistrationConfig& config) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    double t[12];
    to12(initial, t);
    const kreg_b200::Registration r =
        kreg_b200::register_clouds(E.context(), E.cloud(X), E.cloud(Z), t, to_params(params), to_config(config));
    RegistrationResult out;
    out.transform = from12(r.transform);
    out.converged = r.converged;
    out.iterations = r.iterations;
    out.objective_trace = r.objective;
    out.indicator_trace = r.indicator;
    out.lengthscale_trace = r.lengthscale;
    out.step_trace = r.step;
    out.twist_norm_trace = r.twist_norm;
    out.pair_count_trace = r.pair_count;
    out.rebuild_trace = r.rebuild;
    out.final_indicator = r.final_indicator;
    return out;
  });
}

SequenceResult register_sequence(std::span<const PointCloud> frames, const KernelParams& params,
                                 const RegistrationConfig& config) {
  return translate([&] {
    Engine& E = engine();
    std::lock_guard<std::mutex> lk(E.mu);
    // frames are uploaded for this call only (not cached: a long sequence
    // would evict every other cloud)
    std::vector<std::unique_ptr<kreg_b200::Cloud>> up;
    std::vector<const kreg_cloud*> handles;
    for (const PointCloud& f : frames) {
      up.push_back(std::make_unique<kreg_b200::Cloud>(E.context(), view_of(f)));
      handles.push_back(up.back()->get());
    }
    const kreg_b200::Sequence s = kreg_b200::register_sequence(E.context(), handles, to_params(params),
                                                               to_config(config));
    SequenceResult out;
    const size_t n = frames.size(), m = n > 0 ? n - 1 : 0;
    for (size_t k = 0; k < m; ++k) out.relative.push_back(from12(s.relative.data() + 12 * k));
    for (size_t k = 0; k < n; ++k) out.trajectory.push_back(from12(s.trajectory.data() + 12 * k));
    out.fallback = s.fallback;
    out.converged = s.converged;
    out.final_indicator = s.final_indicator;
    out.iterations.assign(s.iterations.begin(), s.iterations.end());
    return out;
  });
}

}  // namespace kreg
