// TEST INFRASTRUCTURE — C-ABI shim over the UNMODIFIED reference library.
//
// The reference's hot-path sources are compiled in place from
// /root/reference/proj/src by oracle/Makefile (against the test-only Eigen
// shim) into oracle/_ref/libkreg_ref.so together with this file. This file
// only marshals the same POD descriptors as include/kreg_b200.h into the
// reference's own C++ API (kreg::build_pairs, kreg::register_clouds, ...),
// so the parity tests and the CPU baseline can call the real reference.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load it.

#include <omp.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "kreg/cloud_io.hpp"
#include "kreg/errors.hpp"
#include "kreg/eval.hpp"
#include "kreg/image.hpp"
#include "kreg/projection.hpp"
#include "kreg/selector.hpp"
#include "kreg/inner_product.hpp"
#include "kreg/reference.hpp"
#include "kreg/registration.hpp"
#include "kreg_b200.h"

using namespace kreg;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const NoOverlapError& e) {
    return fail(KREG_NO_OVERLAP, e.what());
  } catch (const ParseError& e) {
    return fail(KREG_PARSE_ERROR, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(KREG_INVALID_ARGUMENT, e.what());
  } catch (const std::exception& e) {
    return fail(KREG_RUNTIME_ERROR, e.what());
  }
}

PointCloud to_cloud(const kreg_cloud_view* v) {
  std::vector<Eigen::Vector3d> pos(static_cast<size_t>(v->n));
  for (int i = 0; i < v->n; ++i) {
    pos[static_cast<size_t>(i)] = Eigen::Vector3d(v->xyz[3 * i], v->xyz[3 * i + 1], v->xyz[3 * i + 2]);
  }
  if (v->n_channels == 0) return PointCloud(std::move(pos));
  std::vector<Channel> chans;
  for (int k = 0; k < v->n_channels; ++k) {
    chans.push_back({v->channels[k].name, v->channels[k].dim,
                     static_cast<ChannelKind>(v->channels[k].kind)});
  }
  FeatureSchema schema{chans};
  const size_t nf = static_cast<size_t>(v->n) * static_cast<size_t>(v->dim);
  std::vector<double> feat(v->features, v->features + nf);
  return PointCloud(std::move(pos), std::move(schema), std::move(feat));
}

KernelParams to_params(const kreg_kernel_params* p) {
  KernelParams out;
  out.sigma = p->sigma;
  out.lengthscale = p->lengthscale;
  for (int k = 0; k < p->n_channels; ++k) {
    out.per_channel.push_back({p->per_channel[k].sigma, p->per_channel[k].lengthscale,
                               static_cast<KernelForm>(p->per_channel[k].form)});
  }
  return out;
}

RegistrationConfig to_config(const kreg_registration_config* c) {
  RegistrationConfig r;
  r.init_lengthscale = c->init_lengthscale;
  r.subsequent_lengthscale = c->subsequent_lengthscale;
  r.min_lengthscale = c->min_lengthscale;
  r.decay_factor = c->decay_factor;
  r.stabilization_window = c->stabilization_window;
  r.stabilization_rel_tol = c->stabilization_rel_tol;
  r.max_iterations = c->max_iterations;
  r.step_init = c->step_init;
  r.step_shrink = c->step_shrink;
  r.step_grow = c->step_grow;
  r.max_backtracks = c->max_backtracks;
  r.convergence_twist_norm = c->convergence_twist_norm;
  r.cutoff_multiplier = c->cutoff_multiplier;
  r.c_min = c->c_min;
  return r;
}

Isometry to_iso(const double* t) {
  Isometry T;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) T.rotation(r, c) = t[4 * r + c];
    T.translation[r] = t[4 * r + 3];
  }
  return T;
}

void from_iso(const Isometry& T, double* t) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) t[4 * r + c] = T.rotation(r, c);
    t[4 * r + 3] = T.translation[r];
  }
}

void fill_result(const RegistrationResult& res, kreg_registration_result* out) {
  from_iso(res.transform, out->transform);
  out->converged = res.converged ? 1 : 0;
  out->iterations = res.iterations;
  out->final_indicator = res.final_indicator;
  const int n = std::min(out->trace_capacity, res.iterations);
  for (int i = 0; i < n; ++i) {
    if (out->objective_trace) out->objective_trace[i] = res.objective_trace[static_cast<size_t>(i)];
    if (out->indicator_trace) out->indicator_trace[i] = res.indicator_trace[static_cast<size_t>(i)];
    if (out->lengthscale_trace) out->lengthscale_trace[i] = res.lengthscale_trace[static_cast<size_t>(i)];
    if (out->step_trace) out->step_trace[i] = res.step_trace[static_cast<size_t>(i)];
    if (out->twist_norm_trace) out->twist_norm_trace[i] = res.twist_norm_trace[static_cast<size_t>(i)];
    if (out->pair_count_trace) out->pair_count_trace[i] = res.pair_count_trace[static_cast<size_t>(i)];
    if (out->rebuild_trace) out->rebuild_trace[i] = res.rebuild_trace[static_cast<size_t>(i)];
  }
  out->sweeps = 0;
  out->rebuilds = 0;
}

struct RefPairs {
  PairList pairs;
};

}  // namespace

extern "C" {

const char* kref_last_error(void) { return g_err.c_str(); }

void kref_set_threads(int n) { omp_set_num_threads(n); }
int kref_max_threads(void) { return omp_get_max_threads(); }

int kref_build_pairs(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                     const kreg_kernel_params* params, double cutoff_multiplier, double c_min,
                     int dense, void** out, int64_t* n_pairs) {
  return guarded([&] {
    const PointCloud x = to_cloud(X), z = to_cloud(Z);
    auto* p = new RefPairs;
    p->pairs = dense ? reference::dense_pairs(x, z, to_iso(T), to_params(params), cutoff_multiplier, c_min)
                     : build_pairs(x, z, to_iso(T), to_params(params), cutoff_multiplier, c_min);
    *n_pairs = p->pairs.size();
    *out = p;
  });
}

void kref_pairs_destroy(void* p) { delete static_cast<RefPairs*>(p); }

void kref_pairs_export(const void* handle, int64_t* offsets, int32_t* x_index, double* coeff) {
  const PairList& p = static_cast<const RefPairs*>(handle)->pairs;
  std::memcpy(offsets, p.offsets.data(), p.offsets.size() * sizeof(int64_t));
  std::memcpy(x_index, p.x_index.data(), p.x_index.size() * sizeof(int32_t));
  std::memcpy(coeff, p.coeff.data(), p.coeff.size() * sizeof(double));
}

// mode 0: parallel engine objective_and_gradient; 1: serial reference lane
int kref_objective_and_gradient(const void* handle, const kreg_cloud_view* X,
                                const kreg_cloud_view* Z, const double T[12],
                                const kreg_kernel_params* params, int serial, double out[7]) {
  return guarded([&] {
    const PairList& p = static_cast<const RefPairs*>(handle)->pairs;
    const PointCloud x = to_cloud(X), z = to_cloud(Z);
    const Evaluation ev = serial
                              ? reference::pruned_objective_and_gradient(p, x, z, to_iso(T), to_params(params))
                              : objective_and_gradient(p, x, z, to_iso(T), to_params(params));
    out[0] = ev.value;
    for (int k = 0; k < 3; ++k) {
      out[1 + k] = ev.grad.omega[k];
      out[4 + k] = ev.grad.v[k];
    }
  });
}

int kref_inner_product(const void* handle, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                       const double T[12], const kreg_kernel_params* params, double* value) {
  return guarded([&] {
    const PairList& p = static_cast<const RefPairs*>(handle)->pairs;
    *value = inner_product(p, to_cloud(X), to_cloud(Z), to_iso(T), to_params(params));
  });
}

int kref_dense_inner_product(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                             const kreg_kernel_params* params, double* value) {
  return guarded([&] {
    *value = reference::dense_inner_product(to_cloud(X), to_cloud(Z), to_iso(T), to_params(params));
  });
}

int kref_max_point_displacement(const kreg_cloud_view* Z, const double built[12],
                                const double now[12], double* value) {
  return guarded([&] { *value = max_point_displacement(to_cloud(Z), to_iso(built), to_iso(now)); });
}

int kref_indicator(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                   const kreg_kernel_params* params, double cutoff_multiplier, double c_min,
                   double* value) {
  return guarded([&] {
    *value = indicator(to_cloud(X), to_cloud(Z), to_iso(T), to_params(params), cutoff_multiplier, c_min);
  });
}

int kref_exact_cosine(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                      const kreg_kernel_params* params, double* value) {
  return guarded([&] { *value = exact_cosine(to_cloud(X), to_cloud(Z), to_iso(T), to_params(params)); });
}

int kref_register_clouds(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double initial[12],
                         const kreg_kernel_params* params, const kreg_registration_config* config,
                         kreg_registration_result* result) {
  return guarded([&] {
    const RegistrationResult res = register_clouds(to_cloud(X), to_cloud(Z), to_iso(initial),
                                                   to_params(params), to_config(config));
    fill_result(res, result);
  });
}

// Throughput mode: independent registrations, OpenMP over pairs with one
// thread each (nested regions run single-threaded), as synth_bench does
// (reference eval.cpp:323). Clouds are converted before the timed loop.
int kref_register_batch(int n, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                        const double* initials, const kreg_kernel_params* params,
                        const kreg_registration_config* config, kreg_registration_result* results,
                        int* statuses, double* seconds) {
  return guarded([&] {
    std::vector<PointCloud> xs, zs;
    for (int k = 0; k < n; ++k) {
      xs.push_back(to_cloud(&X[k]));
      zs.push_back(to_cloud(&Z[k]));
    }
    const KernelParams kp = to_params(params);
    const RegistrationConfig rc = to_config(config);
    const double t0 = omp_get_wtime();
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < n; ++k) {
      try {
        const RegistrationResult res =
            register_clouds(xs[static_cast<size_t>(k)], zs[static_cast<size_t>(k)],
                            to_iso(initials + 12 * k), kp, rc);
        fill_result(res, &results[k]);
        statuses[k] = 0;
      } catch (const NoOverlapError&) {
        statuses[k] = KREG_NO_OVERLAP;
      } catch (const std::invalid_argument&) {
        statuses[k] = KREG_INVALID_ARGUMENT;
      } catch (const std::exception&) {
        statuses[k] = KREG_RUNTIME_ERROR;
      }
    }
    *seconds = omp_get_wtime() - t0;
  });
}

int kref_register_sequence(const kreg_cloud_view* frames, int n_frames,
                           const kreg_kernel_params* params, const kreg_registration_config* config,
                           kreg_sequence_result* out) {
  return guarded([&] {
    std::vector<PointCloud> fs;
    for (int k = 0; k < n_frames; ++k) fs.push_back(to_cloud(&frames[k]));
    const SequenceResult seq = register_sequence(fs, to_params(params), to_config(config));
    for (size_t k = 0; k < seq.relative.size(); ++k) {
      from_iso(seq.relative[k], out->relative + 12 * k);
      out->fallback[k] = seq.fallback[k];
      out->converged[k] = seq.converged[k];
      out->final_indicator[k] = seq.final_indicator[k];
      out->iterations[k] = seq.iterations[k];
    }
    for (size_t k = 0; k < seq.trajectory.size(); ++k) from_iso(seq.trajectory[k], out->trajectory + 12 * k);
  });
}

int kref_anneal_step(double lengthscale, const double* history, int n,
                     const kreg_registration_config* config, double* next) {
  return guarded([&] {
    *next = anneal_step(lengthscale, std::span<const double>(history, static_cast<size_t>(n)),
                        to_config(config));
  });
}

int kref_line_search(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                     const double g[6], const kreg_kernel_params* params, const void* handle,
                     const kreg_registration_config* config, double* step) {
  return guarded([&] {
    Twist tw;
    for (int k = 0; k < 3; ++k) {
      tw.omega[k] = g[k];
      tw.v[k] = g[3 + k];
    }
    *step = line_search(to_cloud(X), to_cloud(Z), to_iso(T), tw, to_params(params),
                        static_cast<const RefPairs*>(handle)->pairs, to_config(config));
  });
}

int kref_check_config(const kreg_registration_config* config) {
  return guarded([&] { check_config(to_config(config)); });
}

int kref_se3_exp(const double xi[6], double out[12]) {
  return guarded([&] {
    Twist tw;
    for (int k = 0; k < 3; ++k) {
      tw.omega[k] = xi[k];
      tw.v[k] = xi[3 + k];
    }
    from_iso(kreg::exp(tw), out);
  });
}

void kref_se3_compose(const double a[12], const double b[12], double out[12]) {
  from_iso(compose(to_iso(a), to_iso(b)), out);
}

double kref_diameter(const kreg_cloud_view* v) { return diameter(to_cloud(v)); }

// Cloud file I/O (cloud_io.cpp:141-297 read_ply, 456-529 write_ply).
int kref_write_ply(const kreg_cloud_view* v, const char* path, int binary) {
  return guarded([&] { write_ply(to_cloud(v), path, binary != 0); });
}
// read_ply into a heap PointCloud; *warnings gets the skipped-property lines
int kref_read_ply(const char* path, void** out, int* n, int* dim, int* n_channels, char* warnings, int cap) {
  return guarded([&] {
    std::vector<std::string> w;
    auto* c = new PointCloud(read_cloud(path, &w));
    *out = c;
    *n = c->size();
    *dim = c->schema().total_dim();
    *n_channels = c->schema().channel_count();
    std::string all;
    for (const auto& s : w) all += s + "\n";
    if (warnings && cap > 0) {
      const size_t k = std::min(all.size(), static_cast<size_t>(cap - 1));
      std::memcpy(warnings, all.data(), k);
      warnings[k] = '\0';
    }
  });
}
void kref_cloud_copy(const void* h, double* xyz, double* features, int* dims, int* kinds) {
  const auto* c = static_cast<const PointCloud*>(h);
  for (int i = 0; i < c->size(); ++i) {
    const Eigen::Vector3d& p = c->position(i);
    xyz[3 * i] = p.x();
    xyz[3 * i + 1] = p.y();
    xyz[3 * i + 2] = p.z();
    const auto row = c->feature_row(i);
    for (int d = 0; d < c->schema().total_dim(); ++d) features[static_cast<size_t>(i) * c->schema().total_dim() + d] = row[static_cast<size_t>(d)];
  }
  for (int k = 0; k < c->schema().channel_count(); ++k) {
    dims[k] = c->schema().channel(k).dim;
    kinds[k] = static_cast<int>(c->schema().channel(k).kind);
  }
}
void kref_cloud_destroy(void* h) { delete static_cast<PointCloud*>(h); }

// Generators (reference eval.cpp:248-300), for fixtures.
int kref_make_box_cloud(uint64_t seed, int n, int with_color, double* xyz, double* features) {
  return guarded([&] {
    const PointCloud c = make_box_cloud(seed, n, with_color != 0);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) xyz[3 * i + k] = c.position(i)[k];
    if (with_color) std::memcpy(features, c.features().data(), c.features().size() * sizeof(double));
  });
}

int kref_make_ring_cloud(uint64_t seed, int sectors, int per_sector, int with_color, double* xyz,
                         double* features) {
  return guarded([&] {
    const PointCloud c = make_ring_cloud(seed, sectors, per_sector, with_color != 0);
    for (int i = 0; i < c.size(); ++i)
      for (int k = 0; k < 3; ++k) xyz[3 * i + k] = c.position(i)[k];
    if (with_color) std::memcpy(features, c.features().data(), c.features().size() * sizeof(double));
  });
}

// Frame ingest (selector.cpp / projection.cpp): plain arrays in, the
// reference's Selection / PointCloud out (rows copied when capacity suffices).
namespace {
SelectorConfig to_sel(const kreg_selector_config* s) {
  SelectorConfig o;
  o.target_min = s->target_min;
  o.target_max = s->target_max;
  o.initial_threshold = s->initial_threshold;
  o.adjust_factor = s->adjust_factor;
  o.max_adjust_rounds = s->max_adjust_rounds;
  return o;
}
ImageU8 to_img(const uint8_t* p, int w, int h, int c) {
  ImageU8 im(w, h, c);
  std::memcpy(im.data.data(), p, static_cast<size_t>(w) * h * c);
  return im;
}
}  // namespace

int kref_select_points(const uint8_t* rgb, int channels, int w, int h, const uint8_t* valid,
                       const kreg_selector_config* sel, int32_t* pixels, int64_t cap, kreg_selection_info* info,
                       char* note, int note_cap) {
  return guarded([&] {
    const Selection s = select_points(to_img(rgb, w, h, channels),
                                      std::vector<uint8_t>(valid, valid + static_cast<size_t>(w) * h), to_sel(sel));
    info->count = static_cast<int64_t>(s.pixels.size());
    info->threshold = s.threshold;
    info->in_band = s.in_band ? 1 : 0;
    info->fallback = s.note.find("fallback") != std::string::npos ? 1 : 0;
    info->valid_pixels = 0;
    if (cap >= info->count)
      for (size_t k = 0; k < s.pixels.size(); ++k) {
        pixels[2 * k] = s.pixels[k].first;
        pixels[2 * k + 1] = s.pixels[k].second;
      }
    if (note && note_cap > 0) std::snprintf(note, note_cap, "%s", s.note.c_str());
  });
}

int kref_depth_rgb_to_cloud(const uint16_t* depth, const uint8_t* rgb, int channels, const float* sem, int sem_ch,
                            int w, int h, const kreg_camera_intrinsics* in, const kreg_selector_config* sel,
                            double* xyz, double* feat, int64_t cap, int64_t* n, char* note, int note_cap) {
  return guarded([&] {
    ImageU16 d(w, h, 1);
    std::memcpy(d.data.data(), depth, static_cast<size_t>(w) * h * sizeof(uint16_t));
    ImageF s;
    if (sem) {
      s = ImageF(w, h, sem_ch);
      std::memcpy(s.data.data(), sem, static_cast<size_t>(w) * h * sem_ch * sizeof(float));
    }
    CameraIntrinsics ci;
    ci.fx = in->fx; ci.fy = in->fy; ci.cx = in->cx; ci.cy = in->cy;
    ci.depth_scale = in->depth_scale; ci.max_depth = in->max_depth; ci.skip_top_rows = in->skip_top_rows;
    std::vector<std::string> warnings;
    const PointCloud c = depth_rgb_to_cloud(d, to_img(rgb, w, h, channels), sem ? &s : nullptr, ci, to_sel(sel),
                                            &warnings);
    *n = c.size();
    if (cap >= *n) {
      for (int i = 0; i < c.size(); ++i)
        for (int k = 0; k < 3; ++k) xyz[3 * i + k] = c.position(i)[k];
      std::memcpy(feat, c.features().data(), c.features().size() * sizeof(double));
    }
    if (note && note_cap > 0) std::snprintf(note, note_cap, "%s", warnings.empty() ? "" : warnings[0].c_str());
  });
}

}  // extern "C"

// Reference test-helper generators (tests/test_helpers.hpp), so the Python
// replicas in synth.py can be pinned to them (argument evaluation order of
// the C++ calls included).
#include "test_helpers.hpp"

extern "C" {

// n twists from one SplitMix64 stream: out n x 6 (omega, v)
void kref_random_twists(uint64_t seed, double max_angle, double max_translation, int n, double* out) {
  SplitMix64 rng(seed);
  for (int k = 0; k < n; ++k) {
    const Twist t = test::random_twist(rng, max_angle, max_translation);
    for (int c = 0; c < 3; ++c) {
      out[6 * k + c] = t.omega[c];
      out[6 * k + 3 + c] = t.v[c];
    }
  }
}

int kref_random_labeled_cloud(uint64_t seed, int n, double scale, int with_color, int classes, double* xyz,
                              double* features) {
  return guarded([&] {
    const PointCloud c = test::random_labeled_cloud(seed, n, scale, with_color != 0, classes);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) xyz[3 * i + k] = c.position(i)[k];
    std::memcpy(features, c.features().data(), c.features().size() * sizeof(double));
  });
}

int kref_clustered_cloud(uint64_t seed, int clusters, int per_cluster, double center_box, double radius,
                         int with_color, double* xyz, double* features) {
  return guarded([&] {
    const PointCloud c = test::clustered_cloud(seed, clusters, per_cluster, center_box, radius, with_color != 0);
    for (int i = 0; i < c.size(); ++i)
      for (int k = 0; k < 3; ++k) xyz[3 * i + k] = c.position(i)[k];
    std::memcpy(features, c.features().data(), c.features().size() * sizeof(double));
  });
}

}  // extern "C"
