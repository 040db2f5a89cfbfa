// Host runtime: contexts, cloud upload (Morton-sorted device SoA), pair-list
// workspaces and the batched round executor.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <sstream>
#include <mutex>
#include <thread>

#include "engine_host.hpp"

kreg_ctx::~kreg_ctx() {
  kreg_host::nccl_free(nccl);
  for (cudaEvent_t& e : timer)
    if (e) cudaEventDestroy(e);
  for (kreg_pairs* p : pool) delete p;
  pool.clear();
  for (auto*& S : rs) {
    delete S;
    S = nullptr;
  }
}

namespace kreg_host {

namespace {
thread_local std::string g_last_error;
constexpr long long kMaxCells = 1LL << 24;  // dense grid cap; larger => coarser cells
}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }
const char* last_error() { return g_last_error.c_str(); }

void throw_cuda(cudaError_t e, const char* what) {
  cudaGetLastError();
  const kreg_status code = e == cudaErrorMemoryAllocation ? KREG_OUT_OF_MEMORY
                           : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? KREG_NO_DEVICE
                                                                                          : KREG_CUDA_ERROR;
  throw Error(code, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what);
}

Params to_params(const kreg_kernel_params* p) {
  Params out;
  out.sigma = p->sigma;
  out.lengthscale = p->lengthscale;
  for (int k = 0; k < p->n_channels; ++k) out.per_channel.push_back(p->per_channel[k]);
  return out;
}

static const char* kind_name(int k) {
  switch (k) {
    case KREG_KIND_COLOR: return "color";
    case KREG_KIND_INTENSITY: return "intensity";
    case KREG_KIND_SEMANTIC: return "semantic";
    default: return "custom";
  }
}

std::string describe_schema(const kreg_cloud* c) {
  // point_cloud.cpp:33-43
  if (c->schema.empty()) return "<geometric-only>";
  std::ostringstream os;
  for (size_t k = 0; k < c->schema.size(); ++k) {
    if (k) os << ",";
    os << c->schema[k].name << "(" << kind_name(c->schema[k].kind) << ":" << c->schema[k].dim << ")";
  }
  return os.str();
}

void check_same_schema(const kreg_cloud* X, const kreg_cloud* Z, const char* prefix) {
  // inner_product.cpp:26-33 / registration.cpp:77-82
  bool same = X->schema.size() == Z->schema.size();
  for (size_t k = 0; same && k < X->schema.size(); ++k) {
    same = X->schema[k].name == Z->schema[k].name && X->schema[k].dim == Z->schema[k].dim &&
           X->schema[k].kind == Z->schema[k].kind;
  }
  if (!same) {
    throw Error(KREG_INVALID_ARGUMENT, std::string(prefix) + "schema mismatch: X has " + describe_schema(X) +
                                           ", Z has " + describe_schema(Z));
  }
}

void check_kernel_params(const Params& p, const kreg_cloud* c) {
  // kernels.cpp:70-95
  if (!(p.lengthscale > 0.0))
    throw Error(KREG_INVALID_ARGUMENT,
                "kernel params: geometric lengthscale must be > 0, got " + std::to_string(p.lengthscale));
  if (!(p.sigma > 0.0)) throw Error(KREG_INVALID_ARGUMENT, "kernel params: sigma must be > 0");
  if (p.per_channel.size() != c->schema.size()) {
    std::ostringstream os;
    os << "kernel params: " << p.per_channel.size() << " channel entries for schema " << describe_schema(c);
    throw Error(KREG_INVALID_ARGUMENT, os.str());
  }
  for (size_t k = 0; k < p.per_channel.size(); ++k) {
    const kreg_channel_params& cp = p.per_channel[k];
    if (cp.form == KREG_FORM_SQUARED_EXPONENTIAL && !(cp.lengthscale > 0.0))
      throw Error(KREG_INVALID_ARGUMENT,
                  "kernel params: lengthscale of channel '" + c->schema[k].name + "' must be > 0");
    if (!(cp.sigma > 0.0))
      throw Error(KREG_INVALID_ARGUMENT, "kernel params: sigma of channel '" + c->schema[k].name + "' must be > 0");
  }
  if (p.per_channel.size() > static_cast<size_t>(kreg_dev::kMaxChannels))
    throw Error(KREG_INVALID_ARGUMENT, "kernel params: at most 8 feature channels are supported");
}

void check_config(const kreg_registration_config& c) {
  // registration.cpp:12-34
  auto fail = [](const std::string& what) { throw Error(KREG_INVALID_ARGUMENT, "config: " + what); };
  if (!(c.decay_factor > 0.0 && c.decay_factor < 1.0))
    fail("decay_factor must lie in (0, 1), got " + std::to_string(c.decay_factor));
  if (!(c.min_lengthscale > 0.0)) fail("min_lengthscale must be > 0");
  if (!(c.min_lengthscale <= c.init_lengthscale)) fail("min_lengthscale must not exceed init_lengthscale");
  if (!(c.subsequent_lengthscale > 0.0)) fail("subsequent_lengthscale must be > 0");
  if (c.max_iterations < 1) fail("max_iterations must be >= 1");
  if (c.stabilization_window < 1) fail("stabilization_window must be >= 1");
  if (!(c.stabilization_rel_tol > 0.0)) fail("stabilization_rel_tol must be > 0");
  if (!(c.step_init > 0.0)) fail("step_init must be > 0");
  if (!(c.step_shrink > 0.0 && c.step_shrink < 1.0)) fail("step_shrink must lie in (0, 1)");
  if (!(c.step_grow >= 1.0)) fail("step_grow must be >= 1");
  if (c.max_backtracks < 0) fail("max_backtracks must be >= 0");
  if (!(c.convergence_twist_norm > 0.0)) fail("convergence_twist_norm must be > 0");
  if (!(c.cutoff_multiplier >= 1.0)) fail("cutoff_multiplier must be >= 1");
  if (c.c_min < 0.0 || c.c_min >= 1.0) fail("c_min must lie in [0, 1)");
}

double diameter_host(const double* xyz, int n) {
  // point_cloud.cpp:69-87
  if (n <= 1) return 0.0;
  if (n <= 2000) {
    double best = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        const double dx = xyz[3 * i] - xyz[3 * j], dy = xyz[3 * i + 1] - xyz[3 * j + 1],
                     dz = xyz[3 * i + 2] - xyz[3 * j + 2];
        best = std::max(best, dx * dx + dy * dy + dz * dz);
      }
    return std::sqrt(best);
  }
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) lo[k] = hi[k] = xyz[k];
  for (int i = 1; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], xyz[3 * i + k]);
      hi[k] = std::max(hi[k], xyz[3 * i + k]);
    }
  const double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
  return std::sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}

static uint64_t spread3(uint64_t v) {
  v &= 0x1FFFFF;
  v = (v | v << 32) & 0x1F00000000FFFFULL;
  v = (v | v << 16) & 0x1F0000FF0000FFULL;
  v = (v | v << 8) & 0x100F00F00F00F00FULL;
  v = (v | v << 4) & 0x10C30C30C30C30C3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

// Validation + metadata (schema, padded device row layout, diameter, bbox).
kreg_cloud* cloud_describe(kreg_ctx* ctx, const kreg_cloud_view* v) {
  if (v->n < 0) throw Error(KREG_INVALID_ARGUMENT, "PointCloud: negative point count");
  int total = 0;
  for (int k = 0; k < v->n_channels; ++k) {
    if (v->channels[k].dim <= 0)
      throw Error(KREG_INVALID_ARGUMENT, std::string("FeatureSchema: channel '") + v->channels[k].name +
                                             "' has non-positive dim");
    for (int k2 = 0; k2 < k; ++k2)
      if (std::strcmp(v->channels[k].name, v->channels[k2].name) == 0)
        throw Error(KREG_INVALID_ARGUMENT,
                    std::string("FeatureSchema: duplicate channel name '") + v->channels[k].name + "'");
    total += v->channels[k].dim;
  }
  if (total != v->dim) {
    std::ostringstream os;
    os << "PointCloud: feature block has " << static_cast<long long>(v->n) * v->dim << " values, schema with "
       << v->n << " points requires " << static_cast<long long>(v->n) * total;
    throw Error(KREG_INVALID_ARGUMENT, os.str());
  }
  auto c = std::make_unique<kreg_cloud>();
  c->ctx = ctx;
  c->n = v->n;
  c->dim = total;
  // device rows: every channel 16-B aligned and zero-padded to 4k floats
  int padded = 0;
  for (int k = 0; k < v->n_channels; ++k) {
    c->schema.push_back({v->channels[k].name, v->channels[k].dim, v->channels[k].kind});
    c->chan_off.push_back(padded);
    padded += (v->channels[k].dim + 3) / 4 * 4;
  }
  c->fstride = padded;
  if (padded > 64) throw Error(KREG_INVALID_ARGUMENT, "PointCloud: padded feature row > 64 floats is not supported");
  c->diam = diameter_host(v->xyz, v->n);
  if (v->n > 0) {
    for (int k = 0; k < 3; ++k) c->lo[k] = c->hi[k] = v->xyz[k];
    for (int i = 1; i < v->n; ++i)
      for (int k = 0; k < 3; ++k) {
        c->lo[k] = std::min(c->lo[k], v->xyz[3 * i + k]);
        c->hi[k] = std::max(c->hi[k], v->xyz[3 * i + k]);
      }
  }
  return c.release();
}

// Host staging: spatial (Morton) order so that index locality is spatial
// locality; SoA FP64 positions and padded FP32 feature rows written to
// sx/sy/sz/sf (n, n, n, n * fstride elements; pinned memory for fast DMA).
void cloud_stage(const kreg_cloud_view* v, kreg_cloud* c, double* sx, double* sy, double* sz, float* sf) {
  const int n = v->n;
  std::vector<std::pair<uint64_t, int>> keys(static_cast<size_t>(n));
  double span = 0.0;
  for (int k = 0; k < 3; ++k) span = std::max(span, c->hi[k] - c->lo[k]);
  const double s = span > 0 ? (double)((1 << 21) - 1) / span : 0.0;
  for (int i = 0; i < n; ++i) {
    uint64_t m = 0;
    for (int k = 0; k < 3; ++k) {
      const double f = (v->xyz[3 * i + k] - c->lo[k]) * s;
      const uint64_t q = std::isfinite(f) ? static_cast<uint64_t>(std::min(std::max(f, 0.0), 2097151.0)) : 0;
      m |= spread3(q) << k;
    }
    keys[static_cast<size_t>(i)] = {m, i};
  }
  // stable LSD radix sort on the 63-bit key (6 passes of 11 bits): the order
  // of std::sort on (key, index) pairs, in O(n)
  {
    std::vector<std::pair<uint64_t, int>> tmp(keys.size());
    std::vector<uint32_t> hist(2048);
    for (int pass = 0; pass < 6; ++pass) {
      const int sh = 11 * pass;
      std::fill(hist.begin(), hist.end(), 0u);
      for (const auto& kv : keys) ++hist[(kv.first >> sh) & 2047u];
      uint32_t run = 0;
      for (uint32_t& h : hist) {
        const uint32_t c = h;
        h = run;
        run += c;
      }
      for (const auto& kv : keys) tmp[hist[(kv.first >> sh) & 2047u]++] = kv;
      keys.swap(tmp);
    }
  }
  c->order.resize(static_cast<size_t>(n));
  c->rank.resize(static_cast<size_t>(n));
  std::vector<int> src_off;
  int so = 0;
  for (int k = 0; k < v->n_channels; ++k) {
    src_off.push_back(so);
    so += v->channels[k].dim;
  }
  const int fs = c->fstride, dim = c->dim;
  for (int r = 0; r < n; ++r) {
    const int i = keys[static_cast<size_t>(r)].second;
    c->order[static_cast<size_t>(r)] = i;
    c->rank[static_cast<size_t>(i)] = r;
    sx[r] = v->xyz[3 * i];
    sy[r] = v->xyz[3 * i + 1];
    sz[r] = v->xyz[3 * i + 2];
    float* row = sf + static_cast<size_t>(r) * fs;
    for (int d = 0; d < fs; ++d) row[d] = 0.0f;
    for (int k = 0; k < v->n_channels; ++k)
      for (int d = 0; d < v->channels[k].dim; ++d)
        row[c->chan_off[k] + d] = static_cast<float>(v->features[static_cast<size_t>(i) * dim + src_off[k] + d]);
  }
}

size_t cloud_stage_doubles(const kreg_cloud* c) { return 3 * static_cast<size_t>(c->n); }
size_t cloud_stage_floats(const kreg_cloud* c) { return static_cast<size_t>(c->n) * c->fstride + 4; }

// Device copies (async on the context stream) into dx/dy/dz/df, or into
// buffers owned by the cloud when dx == nullptr.
void cloud_upload(kreg_ctx* ctx, kreg_cloud* c, const double* sx, const double* sy, const double* sz, const float* sf,
                  double* dx, double* dy, double* dz, float* df, double4* dw) {
  const int n = c->n;
  if (dx) {
    c->x.borrow(dx, n);
    c->y.borrow(dy, n);
    c->z.borrow(dz, n);
    c->feat.borrow(df, cloud_stage_floats(c));
    c->xw.borrow(dw, static_cast<size_t>(n) + 1);
  } else {
    c->x.ensure(n, false, 1.0);
    c->y.ensure(n, false, 1.0);
    c->z.ensure(n, false, 1.0);
    c->feat.ensure(cloud_stage_floats(c), false, 1.0);
    c->xw.ensure(static_cast<size_t>(n) + 1, false, 1.0);
  }
  if (n) {
    ctx->h2d_bytes += static_cast<long long>(sizeof(double) * 3 * n + sizeof(float) * static_cast<size_t>(n) * c->fstride);
    KREG_CUDA(cudaMemcpyAsync(c->x.ptr, sx, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(c->y.ptr, sy, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(c->z.ptr, sz, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    if (c->fstride)
      KREG_CUDA(cudaMemcpyAsync(c->feat.ptr, sf, sizeof(float) * static_cast<size_t>(n) * c->fstride,
                                cudaMemcpyHostToDevice, ctx->stream));
    kreg_dev::interleave_positions(c->x.ptr, c->y.ptr, c->z.ptr, n, c->xw.ptr, ctx->stream);
  }
}

kreg_cloud* cloud_create(kreg_ctx* ctx, const kreg_cloud_view* v) {
  std::unique_ptr<kreg_cloud> c(cloud_describe(ctx, v));
  KREG_CUDA(cudaSetDevice(ctx->device));
  std::vector<double> h(cloud_stage_doubles(c.get()));
  std::vector<float> f(cloud_stage_floats(c.get()));
  const int n = c->n;
  cloud_stage(v, c.get(), h.data(), h.data() + n, h.data() + 2 * n, f.data());
  cloud_upload(ctx, c.get(), h.data(), h.data() + n, h.data() + 2 * n, f.data(), nullptr, nullptr, nullptr, nullptr,
               nullptr);
  KREG_CUDA(cudaStreamSynchronize(ctx->stream));  // host staging vectors go out of scope
  return c.release();
}

// Many clouds at once (end-to-end calls): validation and staging run on host
// worker threads into pinned context memory, device copies go into one
// context arena (no per-cloud allocation), all on the context stream.
std::vector<std::unique_ptr<kreg_cloud>> cloud_create_many(kreg_ctx* ctx, const kreg_cloud_view* const* views,
                                                           int n) {
  using clk = std::chrono::steady_clock;
  const auto t_begin = clk::now();
  std::vector<std::unique_ptr<kreg_cloud>> out(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) out[k].reset(cloud_describe(ctx, views[k]));
  std::vector<size_t> doff(static_cast<size_t>(n) + 1, 0), foff(static_cast<size_t>(n) + 1, 0),
      woff(static_cast<size_t>(n) + 1, 0);
  for (int k = 0; k < n; ++k) {
    doff[k + 1] = doff[k] + (cloud_stage_doubles(out[k].get()) + 1) / 2 * 2;  // 16-B aligned slices
    foff[k + 1] = foff[k] + (cloud_stage_floats(out[k].get()) + 3) / 4 * 4;
    woff[k + 1] = woff[k] + static_cast<size_t>(out[k]->n) + 1;
  }
  KREG_CUDA(cudaSetDevice(ctx->device));
  KREG_CUDA(cudaStreamSynchronize(ctx->stream));  // staging / arena may still be in use
  ctx->stage_d.ensure(doff[n] + 2);
  ctx->stage_f.ensure(foff[n] + 4);
  ctx->arena_d.ensure(doff[n] + 2, false, 1.25);
  ctx->arena_f.ensure(foff[n] + 4, false, 1.25);
  ctx->arena_w.ensure(woff[n] + 1, false, 1.25);
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int workers = static_cast<int>(std::min<unsigned>(std::min<unsigned>(hw, 32u), static_cast<unsigned>(n)));
  std::vector<std::exception_ptr> err(static_cast<size_t>(std::max(workers, 1)));
  auto work = [&](int w) {
    try {
      for (int k = w; k < n; k += workers) {
        const int m = out[k]->n;
        double* d = ctx->stage_d.ptr + doff[k];
        cloud_stage(views[k], out[k].get(), d, d + m, d + 2 * m, ctx->stage_f.ptr + foff[k]);
      }
    } catch (...) {
      err[static_cast<size_t>(w)] = std::current_exception();
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w) pool.emplace_back(work, w);
  if (workers > 0) work(0);
  for (auto& t : pool) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  const auto t_staged = clk::now();
  for (int k = 0; k < n; ++k) {
    const int m = out[k]->n;
    const double* d = ctx->stage_d.ptr + doff[k];
    double* a = ctx->arena_d.ptr + doff[k];
    cloud_upload(ctx, out[k].get(), d, d + m, d + 2 * m, ctx->stage_f.ptr + foff[k], a, a + m, a + 2 * m,
                 ctx->arena_f.ptr + foff[k], ctx->arena_w.ptr + woff[k]);
  }
  ctx->t_stage += std::chrono::duration<double>(t_staged - t_begin).count();
  ctx->t_upload_issue += std::chrono::duration<double>(clk::now() - t_staged).count();
  return out;
}

// Asynchronous variant for end-to-end batches: cloud pairs (2k, 2k + 1) are
// staged and their copies enqueued on the context stream by worker threads in
// job order; ready[k] turns 1 once job k's copies are enqueued (the solver
// starts job k only then, so stream order puts the copies first).
AsyncUpload::~AsyncUpload() {
  for (auto& t : workers)
    if (t.joinable()) t.join();
  for (cudaEvent_t e : done)
    if (e) cudaEventDestroy(e);
}

std::unique_ptr<AsyncUpload> cloud_upload_async(kreg_ctx* ctx, const kreg_cloud_view* const* views, int n_jobs,
                                                int per_unit, std::vector<int> order) {
  if (order.size() != static_cast<size_t>(n_jobs)) {
    order.resize(static_cast<size_t>(n_jobs));
    for (int j = 0; j < n_jobs; ++j) order[static_cast<size_t>(j)] = j;
  }
  auto ord = std::make_shared<std::vector<int>>(std::move(order));
  auto up = std::make_unique<AsyncUpload>();
  const int n = per_unit * n_jobs;
  up->clouds.resize(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) up->clouds[k].reset(cloud_describe(ctx, views[k]));
  std::vector<size_t> doff(static_cast<size_t>(n) + 1, 0), foff(static_cast<size_t>(n) + 1, 0),
      woff(static_cast<size_t>(n) + 1, 0);
  for (int k = 0; k < n; ++k) {
    doff[k + 1] = doff[k] + (cloud_stage_doubles(up->clouds[k].get()) + 1) / 2 * 2;
    foff[k + 1] = foff[k] + (cloud_stage_floats(up->clouds[k].get()) + 3) / 4 * 4;
    woff[k + 1] = woff[k] + static_cast<size_t>(up->clouds[k]->n) + 1;
  }
  KREG_CUDA(cudaSetDevice(ctx->device));
  KREG_CUDA(cudaStreamSynchronize(ctx->stream));  // staging / arena may still be in use
  ctx->stage_d.ensure(doff[n] + 2);
  ctx->stage_f.ensure(foff[n] + 4);
  ctx->arena_d.ensure(doff[n] + 2, false, 1.25);
  ctx->arena_f.ensure(foff[n] + 4, false, 1.25);
  ctx->arena_w.ensure(woff[n] + 1, false, 1.25);
  up->ready = std::vector<std::atomic<int>>(static_cast<size_t>(n_jobs));
  up->done.assign(static_cast<size_t>(n_jobs), nullptr);
  for (auto& e : up->done) KREG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& r : up->ready) r.store(0);
  const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
  // staging threads (the solver thread keeps a core); KREG_STAGE_WORKERS overrides
  unsigned cap = std::min(hw - 1, 31u);
  if (const char* e = std::getenv("KREG_STAGE_WORKERS")) cap = std::max(1, std::atoi(e));
  const int workers = static_cast<int>(std::min<unsigned>(cap, static_cast<unsigned>(n_jobs)));
  auto next = std::make_shared<std::atomic<int>>(0);
  AsyncUpload* U = up.get();
  const int device = ctx->device;
  auto work = [U, ctx, views, doff, foff, woff, next, n_jobs, per_unit, device, ord]() {
    cudaSetDevice(device);
    for (;;) {
      const int pos = next->fetch_add(1);
      if (pos >= n_jobs) return;
      const int job = (*ord)[static_cast<size_t>(pos)];
      try {
        for (int h = 0; h < per_unit; ++h) {
          const int k = per_unit * job + h;
          kreg_cloud* c = U->clouds[k].get();
          const int m = c->n;
          double* d = ctx->stage_d.ptr + doff[k];
          cloud_stage(views[k], c, d, d + m, d + 2 * m, ctx->stage_f.ptr + foff[k]);
          double* a = ctx->arena_d.ptr + doff[k];
          cloud_upload(ctx, c, d, d + m, d + 2 * m, ctx->stage_f.ptr + foff[k], a, a + m, a + 2 * m,
                       ctx->arena_f.ptr + foff[k], ctx->arena_w.ptr + woff[k]);
        }
        KREG_CUDA(cudaEventRecord(U->done[static_cast<size_t>(job)], ctx->stream));
        U->ready[job].store(1, std::memory_order_release);
      } catch (...) {
        {
          std::lock_guard<std::mutex> lk(U->mu);
          if (!U->error) U->error = std::current_exception();
        }
        U->ready[job].store(-1, std::memory_order_release);
      }
    }
  };
  for (int w = 0; w < workers; ++w) up->workers.emplace_back(work);
  return up;
}

// ------------------------------------------------------------ build setup
static void fill_coeff_params(const BuildJob& job, const kreg_cloud* X, kreg_dev::CoeffParams& cp) {
  // kernels.cpp:18-53; c_ij does not depend on the geometric lengthscale, so
  // a candidate list stays valid across annealing levels
  std::memset(&cp, 0, sizeof(cp));
  cp.n_channels = static_cast<int>(job.params.per_channel.size());
  cp.fstride = X->fstride;
  cp.c_min = static_cast<float>(job.c_min);
  for (int k = 0; k < cp.n_channels; ++k) {
    const kreg_channel_params& pc = job.params.per_channel[static_cast<size_t>(k)];
    kreg_dev::ChannelDev& ch = cp.ch[k];
    ch.offset = X->chan_off[static_cast<size_t>(k)];
    ch.dim = X->schema[static_cast<size_t>(k)].dim;
    ch.linear = pc.form == KREG_FORM_LINEAR ? 1 : 0;
    ch.kappa = static_cast<float>(-1.4426950408889634 / (2.0 * pc.lengthscale * pc.lengthscale));
    ch.sigma2 = static_cast<float>(pc.sigma * pc.sigma);
  }
}

static void prepare_build(kreg_ctx* ctx, BuildJob& job, kreg_dev::BuildReq& R) {
  kreg_pairs* p = job.pairs;
  const kreg_cloud* X = job.X;
  const kreg_cloud* Z = job.Z;
  std::memset(&R, 0, sizeof(R));
  fill_coeff_params(job, X, R.cp);
  const double cutoff = job.cutoff_multiplier * job.params.lengthscale;

  // Reuse the resident candidate list when it provably contains every pair
  // of the new list: max_j |T z_j - Ts z_j| <= sup_disp + disp_hint (triangle
  // inequality over the list being replaced) and that must fit in R_s - cutoff.
  // ... and while it is not much larger than a fresh one: annealing shrinks
  // the cutoff, so a list kept from a larger lengthscale makes every filter
  // scan (R_s / R_s,new)^3 times the entries (first-frame schedule: 0.95 ->
  // 0.0475); above ctx->sup_shrink the grid is searched again
  const double margin = 1e-9 * p->sup_radius;
  const double fresh = cutoff * (1.0 + std::max(0.0, ctx->skin));
  const double grow = p->sup_radius / fresh;
  const bool reuse = !job.force_full && ctx->skin > 0.0 && p->sup_valid && p->sup_X == X && p->sup_Z == Z &&
                     std::memcmp(&p->sup_cp, &R.cp, sizeof(R.cp)) == 0 && job.disp_hint >= 0.0 &&
                     p->sup_disp + job.disp_hint + cutoff <= p->sup_radius - 2.0 * margin &&
                     grow * grow * grow <= ctx->sup_shrink;
  // ... and the resident sweep list, filtered from that candidate list at
  // T_build with the old cutoff, holds every pair of the new list when
  // max_j |T z_j - T_build z_j| + cutoff <= old cutoff (annealing shrinks the
  // cutoff; guard: FP32 rounding of the two predicates). Checked in-kernel.
  const double guard = 1e-5 * p->cutoff_radius;
  const double sub_limit = p->cutoff_radius - cutoff - guard;
  const bool refilter = reuse && ctx->refilter && !job.no_refilter && p->counts_valid && p->slots > 0 &&
                        p->n_tiles == (Z->n + 31) / 32 && job.disp_hint <= sub_limit;
  double old_T[12];
  std::memcpy(old_T, p->T_build, sizeof(old_T));

  p->ctx = ctx;
  p->X = X;
  p->Z = Z;
  p->built_at_lengthscale = job.params.lengthscale;
  p->cutoff_radius = cutoff;
  p->c_min = job.c_min;
  p->sigma = job.params.sigma;
  p->counts_valid = false;  // until this round's results are read back
  std::memcpy(p->T_build, job.T, sizeof(p->T_build));

  R.xx = X->x.ptr; R.xy = X->y.ptr; R.xz = X->z.ptr; R.xfeat = X->feat.ptr; R.n_x = X->n;
  R.xw = X->xw.ptr;
  R.zx = Z->x.ptr; R.zy = Z->y.ptr; R.zz = Z->z.ptr; R.zfeat = Z->feat.ptr; R.n_z = Z->n;
  std::memcpy(R.T, job.T, sizeof(R.T));
  R.cutoff_sq = cutoff * cutoff;  // inner_product.cpp:59
  const int nx = X->n, nz = Z->n;
  const int n_tiles = (nz + 31) / 32;
  p->n_tiles = n_tiles;
  R.n_tiles = n_tiles;

  if (!reuse) {
    R.full = 1;
    ++ctx->full_builds;
    // why: 0 no resident list, 1 forced (overflow / guard), 2 moved beyond
    // the candidate radius, 3 other (clouds, coefficients, skin)
    const int why = !p->sup_valid ? 0 : job.force_full ? 1
                    : (p->sup_X == X && p->sup_Z == Z && job.disp_hint >= 0.0 && ctx->skin > 0.0 &&
                       std::memcmp(&p->sup_cp, &R.cp, sizeof(R.cp)) == 0) ? (grow * grow * grow > ctx->sup_shrink ? 3 : 2)
                                                                            : 3;
    ++ctx->full_why[why];
    ++p->full_builds;
    const double rs = cutoff * (1.0 + std::max(0.0, ctx->skin));
    p->sup_valid = false;  // until this round's results are read back
    p->sup_X = X;
    p->sup_Z = Z;
    p->sup_cp = R.cp;
    p->sup_radius = rs;
    std::memcpy(p->sup_T, job.T, sizeof(p->sup_T));
    R.sup_cutoff_sq = rs * rs;
    // dense grid over X's bbox; cell >= R_s (margin keeps the 27-cell
    // stencil a superset of the FP64 ball under rounding)
    double h = rs * (1.0 + 1e-7);
    long long g[3];
    for (;;) {
      long long cells = 1;
      for (int k = 0; k < 3; ++k) {
        g[k] = X->n ? static_cast<long long>(std::floor((X->hi[k] - X->lo[k]) / h)) + 1 : 1;
        cells *= g[k];
      }
      if (cells <= kMaxCells) break;
      h *= 1.25;
    }
    for (int k = 0; k < 3; ++k) R.origin[k] = X->lo[k];
    R.inv_h = 1.0 / h;
    R.gx = static_cast<int>(g[0]);
    R.gy = static_cast<int>(g[1]);
    R.gz = static_cast<int>(g[2]);
    R.n_cells = g[0] * g[1] * g[2];
    p->n_cells = R.n_cells;
    p->gx = R.gx; p->gy = R.gy; p->gz = R.gz;
    // grid buffers live in the round's arena (assign_grid_arena): they are
    // only needed by this build's kernels
    const long long want = p->expected_sup > 0 ? p->expected_sup : static_cast<long long>(nz) * 256 + 4096;
    if (p->sup.cap < static_cast<size_t>(want)) {
      p->sup.ensure(static_cast<size_t>(std::max<long long>(want + want / 4, ctx->hw_sup)), false, 1.0);
      p->sup_i.ensure(p->sup.cap, false, 1.0);
      ctx->hw_sup = std::max<long long>(ctx->hw_sup, static_cast<long long>(p->sup.cap));
    }
  } else {
    ++ctx->filter_builds;
    ++p->filter_builds;
  }
  if (refilter) {
    // the current sweep list becomes the source (alt_*), the build writes
    // the other buffer set
    ++ctx->refilter_builds;
    p->alt_slot_buf.ensure(p->slot_buf.cap, false, 1.0);
    p->alt_perm.ensure(p->perm.cap, false, 1.0);
    p->alt_pos.ensure(p->pos.cap, false, 1.0);
    p->alt_deg_s.ensure(p->deg_s.cap, false, 1.0);
    p->alt_tile_off.ensure(p->tile_off.cap, false, 1.0);
    p->alt_unit_off.ensure(p->unit_off.cap, false, 1.0);
    p->alt_zs.ensure(p->zs.cap, false, 1.0);
    p->alt_chunks.ensure(p->chunks.cap, false, 1.0);
    p->slot_buf.swap(p->alt_slot_buf);
    p->perm.swap(p->alt_perm);
    p->pos.swap(p->alt_pos);
    p->deg_s.swap(p->alt_deg_s);
    p->tile_off.swap(p->alt_tile_off);
    p->unit_off.swap(p->alt_unit_off);
    p->zs.swap(p->alt_zs);
    p->chunks.swap(p->alt_chunks);
    R.refilter = 1;
    std::memcpy(R.old_T, old_T, sizeof(R.old_T));
    R.old_slots = p->alt_slot_buf.ptr;
    R.old_perm = p->alt_perm.ptr;
    R.old_deg_s = p->alt_deg_s.ptr;
    R.old_tile_off = p->alt_tile_off.ptr;
    R.old_unit_off = p->alt_unit_off.ptr;
  }
  p->sup_count.ensure(nz + 1);
  p->sup_off.ensure(n_tiles + 2);
  std::memcpy(R.Ts, p->sup_T, sizeof(R.Ts));
  std::memcpy(p->slot_T, p->sup_T, sizeof(p->slot_T));
  R.sup_count = p->sup_count.ptr;
  R.sup_off = p->sup_off.ptr;
  R.sup = p->sup.ptr;
  R.sup_i = p->sup_i.ptr;
  R.sup_capacity = static_cast<long long>(p->sup.cap);
  const double limit = refilter ? sub_limit : p->sup_radius - cutoff - margin;
  R.filter_limit_sq = limit > 0.0 ? limit * limit : 0.0;

  // torque arm origin of the sweep (FP32 arms T z - anchor stay small)
  for (int k = 0; k < 3; ++k) p->anchor[k] = 0.5 * (X->lo[k] + X->hi[k]);

  // sweep-list buffers
  p->count.ensure(nz + 4);
  p->perm.ensure(nz + 1);
  p->pos.ensure(nz + 1);
  p->deg_s.ensure(nz + 1);
  p->zs.ensure(nz + 1);
  p->chunks.ensure(kreg_dev::kMaxChunks + 1);
  R.perm = p->perm.ptr;
  R.pos = p->pos.ptr;
  R.deg_s = p->deg_s.ptr;
  R.zs = p->zs.ptr;
  R.chunks = p->chunks.ptr;
  const long long want = p->expected_pairs > 0 ? p->expected_pairs : static_cast<long long>(nz) * 96 + 4096;
  if (p->slot_buf.cap < static_cast<size_t>(want)) {
    p->slot_buf.ensure(static_cast<size_t>(std::max<long long>(want + want / 2, ctx->hw_slots)), false, 1.0);
    p->slot_i.ensure(p->slot_buf.cap, false, 1.0);
    ctx->hw_slots = std::max<long long>(ctx->hw_slots, static_cast<long long>(p->slot_buf.cap));
  }
  p->tile_off.ensure(n_tiles + 2);
  p->unit_off.ensure(n_tiles + 2);
  p->disp_blk.ensure(nz / 8 + 2);
  R.count = p->count.ptr;
  R.tile_off = p->tile_off.ptr;
  R.unit_off = p->unit_off.ptr;
  R.slots = p->slot_buf.ptr;
  R.slot_i = p->slot_i.ptr;
  R.capacity = static_cast<long long>(p->slot_buf.cap);
  R.disp_blk = p->disp_blk.ptr;
  p->chunk_pref = ctx->chunk_pref;
  R.chunk_pref = p->chunk_pref;
}

// Scratch of request e lives in per-round arenas of the context (several
// requests of one round may sweep the same pair list).
struct SweepScratch {
  size_t part_off = 0;
};

static long long sweep_units(const kreg_pairs* p) {
  // every sweep unit is exactly 32 * kUnitSteps slots (k_tile_offsets)
  return p->slots / (32LL * kreg_dev::kUnitSteps);
}

// chunk partials of one request: at most kMaxChunks x M x (7 | 1) doubles
static size_t sweep_partials(const EvalJob& job) {
  return static_cast<size_t>(kreg_dev::kMaxChunks + kreg_dev::kMaxChunkGroups) * job.M *
         (job.second ? kreg_dev::kNvSecond : job.grad ? 7 : 1);
}

static void prepare_sweep(EvalJob& job, kreg_dev::SweepReq& R, double* partials, unsigned long long* disp_bits) {
  kreg_pairs* p = job.pairs;
  // every field is assigned below; candidate rows m >= M are never read (no
  // memset: ~1.7 KB per request per round on the host's critical path)
  const int nz = p->Z->n;
  R.units = p->counts_valid ? sweep_units(p) : -1;
  R.tile_off = p->tile_off.ptr;
  R.unit_off = p->unit_off.ptr;
  R.zs = p->zs.ptr;
  R.chunks = p->chunks.ptr;
  R.n_tiles = p->n_tiles;
  R.slots = p->slot_buf.ptr;
  R.capacity = static_cast<long long>(p->slot_buf.cap);
  R.grad = job.grad || job.second ? 1 : 0;
  // analytic displacement bound: |(R_m - R_b) z + (t_m - t_b)| <= ||R_m - R_b||_F h + |(R_m - R_b) c + (t_m - t_b)|
  // for z in Z's bounding box (centre c, half-diagonal h)
  job.no_disp = false;
  if (job.disp_limit > 0.0) {
    const kreg_cloud* Zc = p->Z;
    double c[3], h2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      c[k] = 0.5 * (Zc->lo[k] + Zc->hi[k]);
      h2 += 0.25 * (Zc->hi[k] - Zc->lo[k]) * (Zc->hi[k] - Zc->lo[k]);
    }
    const double h = std::sqrt(h2);
    bool all = true;
    for (int m = 0; m < job.M && all; ++m) {
      double fro = 0.0, off2 = 0.0;
      for (int r = 0; r < 3; ++r) {
        double o = job.T[m][4 * r + 3] - p->T_build[4 * r + 3];
        for (int k = 0; k < 3; ++k) {
          const double d = job.T[m][4 * r + k] - p->T_build[4 * r + k];
          fro += d * d;
          o += d * c[k];
        }
        off2 += o * o;
      }
      const double b = (std::sqrt(fro) * h + std::sqrt(off2)) * (1.0 + 1e-9) + 1e-300;
      job.disp_bound[m] = b;
      all = b <= job.disp_limit;
    }
    job.no_disp = all;
    if (p->ctx) {
      ++p->ctx->disp_asked;
      if (all) ++p->ctx->disp_screened;
    }
  }
  R.no_disp = job.no_disp ? 1 : 0;
  R.second = job.second ? 1 : 0;
  if (job.second) {  // u_j = omega x T z_j + v = omega x (arm_j) + (omega x anchor + v)
    const double* w = job.dir;
    const double* a = p->anchor;
    const double v2[3] = {w[1] * a[2] - w[2] * a[1] + w[3], w[2] * a[0] - w[0] * a[2] + w[4],
                          w[0] * a[1] - w[1] * a[0] + w[5]};
    for (int k = 0; k < 3; ++k) {
      R.dir[k] = static_cast<float>(w[k]);
      R.dir[3 + k] = static_cast<float>(v2[k]);
    }
  }
  R.chunk_pref = p->chunk_pref;
  R.zx = p->Z->x.ptr; R.zy = p->Z->y.ptr; R.zz = p->Z->z.ptr;
  R.n_z = nz;
  R.M = job.M;
  for (int m = 0; m < job.M; ++m) std::memcpy(R.T[m], job.T[m], sizeof(double) * 12);
  std::memcpy(R.Tb, p->T_build, sizeof(R.Tb));
  for (int k = 0; k < 3; ++k) R.anchor[k] = p->anchor[k];
  for (int m = 0; m < job.M; ++m) {
    // {R_m - R_s, t_m - t_s} (s: the slots' frame) and {R_m, t_m - anchor}
    // in FP32 (the sweep forms (T_m - T_s) z and T_m z - anchor per source)
    for (int k = 0; k < 12; ++k) {
      R.Td[m][k] = static_cast<float>(job.T[m][k] - p->slot_T[k]);
      R.Ta[m][k] = static_cast<float>(job.T[m][k] - ((k % 4) == 3 ? p->anchor[k / 4] : 0.0));
    }
  }
  const double l = job.lengthscale;
  R.kappa = static_cast<float>(-1.4426950408889634 / (2.0 * l * l));
  R.sigma2 = job.sigma * job.sigma;  // the call's sigma, not the build's (inner_product.cpp:100,126)
  R.inv_l2 = 1.0 / (l * l);
  R.partials = partials;
  R.disp_bits = disp_bits;
}

// Grid buffers of the round's grid searches, carved from one arena per round
// slot (cell counts stay zero between rounds: k_scatter consumes them).
static void assign_grid_arena(RoundSlot& S, kreg_dev::BuildReq* reqs, int nb) {
  size_t cells = 0, pts = 0, tiles = 0, feats = 0;
  for (int b = 0; b < nb; ++b) {
    if (!reqs[b].full) continue;
    feats += static_cast<size_t>(reqs[b].n_x) * reqs[b].cp.fstride + 4;
    cells += static_cast<size_t>(reqs[b].n_cells) + 2;
    pts += static_cast<size_t>(reqs[b].n_x) + 2;
    tiles += static_cast<size_t>(reqs[b].n_cells / kreg_dev::kScanTile) + 4;
  }
  if (!cells) return;
  S.g_count.ensure(cells, /*zero=*/true, 1.5);
  S.g_start.ensure(cells, false, 1.5);
  S.g_int.ensure(3 * pts, false, 1.5);
  S.g_pos.ensure(3 * pts, false, 1.5);
  S.g_scan.ensure(tiles, false, 1.5);
  S.g_feat.ensure(feats + 4, false, 1.5);
  size_t oc = 0, op = 0, ot = 0, of = 0;
  for (int b = 0; b < nb; ++b) {
    kreg_dev::BuildReq& R = reqs[b];
    if (!R.full) continue;
    const size_t np = static_cast<size_t>(R.n_x) + 2;
    R.cell_count = S.g_count.ptr + oc;
    R.cell_start = S.g_start.ptr + oc;
    R.cell_of = S.g_int.ptr + 3 * op;
    R.tmp_items = R.cell_of + np;
    R.cell_items = R.tmp_items + np;
    R.cx = S.g_pos.ptr + 3 * op;
    R.cy = R.cx + np;
    R.cz = R.cy + np;
    R.scan_tiles = S.g_scan.ptr + ot;
    R.cfeat = S.g_feat.ptr + of;  // fstride is a multiple of 4: rows stay 16-B aligned
    of += (static_cast<size_t>(R.n_x) * R.cp.fstride + 3) / 4 * 4;
    oc += static_cast<size_t>(R.n_cells) + 2;
    op += np;
    ot += static_cast<size_t>(R.n_cells / kreg_dev::kScanTile) + 4;
  }
}

RoundSlot* round_slot(kreg_ctx* ctx, int i) {
  if (!ctx->rs[i]) {
    auto* S = new RoundSlot;
    KREG_CUDA(cudaEventCreateWithFlags(&S->done, cudaEventDisableTiming));
    KREG_CUDA(cudaEventCreate(&S->ev0));
    KREG_CUDA(cudaEventCreate(&S->ev1));
    KREG_CUDA(cudaEventCreate(&S->evb0));
    KREG_CUDA(cudaEventCreate(&S->evb1));
    S->stream = ctx->stream;
    if (i == 1 || i >= 3) {
      KREG_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
      KREG_CUDA(cudaEventCreateWithFlags(&S->ordered, cudaEventDisableTiming));
      S->own_stream = true;
    }
    ctx->rs[i] = S;
  }
  return ctx->rs[i];
}

RoundSlot::~RoundSlot() {
  if (done) cudaEventDestroy(done);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (evb0) cudaEventDestroy(evb0);
  if (evb1) cudaEventDestroy(evb1);
  if (ordered) cudaEventDestroy(ordered);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

void begin_round(kreg_ctx* ctx, RoundSlot& S, std::vector<BuildJob>&& builds_in, std::vector<EvalJob>&& evals_in) {
  NvtxScope nvtx("kreg.round.launch");
  S.builds = std::move(builds_in);
  S.evals = std::move(evals_in);
  std::vector<BuildJob>& builds = S.builds;
  std::vector<EvalJob>& evals = S.evals;
  const int nb = static_cast<int>(builds.size());
  const int ne = static_cast<int>(evals.size());
  S.in_flight = false;
  if (nb == 0 && ne == 0) return;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  KREG_CUDA(cudaSetDevice(ctx->device));
  S.h_build.ensure(nb + 1);
  S.d_build.ensure(nb + 1);
  S.h_sweep.ensure(ne + 1);
  S.d_sweep.ensure(ne + 1);
  const size_t n_res = static_cast<size_t>(ne) * kreg_dev::kMaxCandidates * kreg_dev::kOut + kreg_dev::kBuildStatus * (nb + 1);
  S.n_res = n_res;
  // results land in pinned host memory straight from the kernels (UVA maps
  // cudaMallocHost memory into the device address space): no D2H copy, the
  // round's completion event is all the host waits for
  S.h_results.ensure(n_res);

  for (int b = 0; b < nb; ++b) {
    prepare_build(ctx, builds[b], S.h_build.ptr[b]);
    S.h_build.ptr[b].status = S.h_results.ptr + static_cast<size_t>(ne) * kreg_dev::kMaxCandidates * kreg_dev::kOut +
                              kreg_dev::kBuildStatus * b;
  }
  assign_grid_arena(S, S.h_build.ptr, nb);
  for (int b = 0; b < nb; ++b) {
    // (a refilter's list equals the candidate-list filter's: the export
    // re-runs the latter's emit)
    builds[b].pairs->last_req = S.h_build.ptr[b];
    builds[b].pairs->last_req.refilter = 0;
    builds[b].pairs->index_valid = false;
  }
  if (S.own_stream) {  // after the uploads of the clouds this round's first builds read
    for (const BuildJob& bj : builds)
      for (cudaEvent_t e : bj.wait_ev)
        if (e) KREG_CUDA(cudaStreamWaitEvent(S.stream, e, 0));
  }
  // builds go to the device before the sweep requests are prepared
  if (nb) {
    KREG_CUDA(cudaMemcpyAsync(S.d_build.ptr, S.h_build.ptr, sizeof(kreg_dev::BuildReq) * nb, cudaMemcpyHostToDevice,
                              S.stream));
    if (ctx->profiling) KREG_CUDA(cudaEventRecord(S.evb0, S.stream));
    kreg_dev::build_pairs_batched(S.h_build.ptr, S.d_build.ptr, nb, S.stream);
    if (ctx->profiling) KREG_CUDA(cudaEventRecord(S.evb1, S.stream));
  }
  const auto tb = clk::now();
  ctx->t_build_prep += std::chrono::duration<double>(tb - t0).count();
  // F-only requests first (their chunks are the heaviest; see sweep_batched)
  std::stable_partition(evals.begin(), evals.end(), [](const EvalJob& e) { return !e.grad; });
  std::vector<SweepScratch> scratch(static_cast<size_t>(ne));
  size_t part_total = 0;
  for (int e = 0; e < ne; ++e) {
    scratch[e].part_off = part_total;
    part_total += sweep_partials(evals[e]);
  }
  if (ne) {
    S.part_arena.ensure(part_total + 1, false, 1.5);
    S.counter_arena.ensure(kreg_dev::sweep_ctl_bytes(ne) / sizeof(unsigned) + 1, /*zero=*/true);
    S.disp_arena.ensure(static_cast<size_t>(ne + 1) * kreg_dev::kMaxCandidates, /*zero=*/true);
  }
  for (int e = 0; e < ne; ++e) {
    prepare_sweep(evals[e], S.h_sweep.ptr[e], S.part_arena.ptr + scratch[e].part_off,
                  S.disp_arena.ptr + static_cast<size_t>(e) * kreg_dev::kMaxCandidates);
    S.h_sweep.ptr[e].out = S.h_results.ptr + static_cast<size_t>(e) * kreg_dev::kMaxCandidates * kreg_dev::kOut;
  }
  const auto ts = clk::now();
  ctx->t_sweep_prep += std::chrono::duration<double>(ts - tb).count();
  if (ne)
    KREG_CUDA(cudaMemcpyAsync(S.d_sweep.ptr, S.h_sweep.ptr, sizeof(kreg_dev::SweepReq) * ne, cudaMemcpyHostToDevice,
                              S.stream));
  if (ne) {
    S.sweep_issue = ctx->sweep_issued++;
    kreg_dev::sweep_batched(S.h_sweep.ptr, S.d_sweep.ptr, ne, ctx->sm_count, S.counter_arena.ptr, S.stream,
                            ctx->profiling ? S.ev0 : nullptr, ctx->profiling ? S.ev1 : nullptr);
  }
  KREG_CUDA(cudaGetLastError());
  KREG_CUDA(cudaEventRecord(S.done, S.stream));
  S.in_flight = true;
  ctx->t_prepare += std::chrono::duration<double>(clk::now() - t0).count();
}

void end_round(kreg_ctx* ctx, RoundSlot& S) {
  if (!S.in_flight) return;
  NvtxScope nvtx("kreg.round.complete");
  using clk = std::chrono::steady_clock;
  const auto t1 = clk::now();
  KREG_CUDA(cudaEventSynchronize(S.done));
  S.in_flight = false;
  ctx->t_wait += std::chrono::duration<double>(clk::now() - t1).count();
  ctx->rounds += 1;
  std::vector<BuildJob>& builds = S.builds;
  std::vector<EvalJob>& evals = S.evals;
  const int nb = static_cast<int>(builds.size());
  const int ne = static_cast<int>(evals.size());
  const double* res = S.h_results.ptr;
  std::vector<int> redo;
  for (int b = 0; b < nb; ++b) {
    const double* st =
        res + static_cast<size_t>(ne) * kreg_dev::kMaxCandidates * kreg_dev::kOut + kreg_dev::kBuildStatus * b;
    BuildJob& job = builds[b];
    kreg_pairs* p = job.pairs;
    const bool full = S.h_build.ptr[b].full != 0;
    bool ok = true;
    if (full) {
      p->sup_entries = static_cast<long long>(st[4]);
      if (st[3] != 0.0) {  // candidate list overflowed: grow, rebuild from the grid
        p->expected_sup = static_cast<long long>(st[4] * 1.15) + 4096;
        job.force_full = true;
        ok = false;
      } else {
        p->sup_valid = true;
        ctx->hw_radius = std::max(ctx->hw_radius, p->sup_radius);
        p->sup_disp = 0.0;  // built at T: a re-run may filter it
        job.disp_hint = 0.0;
        p->expected_sup = std::max(p->expected_sup, p->sup_entries);
      }
    }
    const bool refilter = S.h_build.ptr[b].refilter != 0;
    if (ok && st[6] != 0.0) {
      if (refilter) {  // the sweep list did not cover the new cutoff: filter the candidate list
        job.no_refilter = true;
      } else {  // candidate radius did not cover the move (rounding guard)
        p->sup_valid = false;
        job.force_full = true;
      }
      ok = false;
    }
    p->P = static_cast<long long>(st[0]);
    p->slots = static_cast<long long>(st[2]);
    if (st[1] != 0.0) {
      p->expected_pairs = static_cast<long long>(st[2] * 1.15) + 1024;
      if (refilter) job.no_refilter = true;
      ok = false;
    } else {
      p->expected_pairs = std::max(p->expected_pairs, p->slots);
    }
    p->counts_valid = ok;
    if (ok) {
      // max_j |T_build z_j - Ts z_j|: measured by a candidate-list filter; a
      // refilter measured |T_build z_j - old T_build z_j| (triangle bound)
      p->sup_disp = refilter ? p->sup_disp + st[5] : st[5];
    } else {
      redo.push_back(b);
    }
  }
  if (!redo.empty()) {
    // grow and re-run the failed builds and every evaluation in this round
    std::vector<BuildJob> b2;
    for (int b : redo) b2.push_back(builds[b]);
    std::vector<EvalJob> e2 = std::move(evals);
    begin_round(ctx, S, std::move(b2), std::move(e2));
    end_round(ctx, S);
    return;
  }
  if (nb && ctx->profiling) {
    float ms = 0.0f;
    KREG_CUDA(cudaEventElapsedTime(&ms, S.evb0, S.evb1));
    ctx->build_ms += ms;
    ctx->build_rounds += 1;
    for (int b = 0; b < nb; ++b) {
      ctx->filter_entries += builds[b].pairs->sup_entries;
      ctx->built_slots += builds[b].pairs->slots;
    }
  }
  long long round_pairs = 0, round_slots = 0;
  long long d2h = static_cast<long long>(sizeof(double)) * kreg_dev::kBuildStatus * nb;  // build statuses
  for (int e = 0; e < ne; ++e) d2h += static_cast<long long>(sizeof(double)) * kreg_dev::kOut * evals[e].M;
  ctx->d2h_bytes += d2h;
  for (int e = 0; e < ne; ++e) {
    std::memcpy(evals[e].out, res + static_cast<size_t>(e) * kreg_dev::kMaxCandidates * kreg_dev::kOut,
                sizeof(double) * (kreg_dev::kOut * evals[e].M + (evals[e].second ? 2 : 0)));
    if (evals[e].no_disp)  // the bound stands in for the maximum (EvalJob::disp_limit)
      for (int m = 0; m < evals[e].M; ++m) evals[e].out[m * kreg_dev::kOut + 7] = evals[e].disp_bound[m];
    ctx->pair_evals += evals[e].pairs->P * evals[e].M;
    round_pairs += evals[e].pairs->P;
    round_slots += evals[e].pairs->slots;
  }
  ctx->pairs_streamed += round_pairs;
  ctx->slots_streamed += round_slots;
  static const bool trace = std::getenv("KREG_TRACE_ROUNDS") != nullptr;
  if (trace && ne)  // diagnostic: match profiled sweep launches to their pair / slot counts
    std::fprintf(stderr, "kreg-round sweeps=%lld launch=%lld requests=%d launches=%d pairs=%lld slots=%lld\n",
                 ctx->sweep_launches, S.sweep_issue, ne, (ne + kreg_dev::kMaxSweepReqs - 1) / kreg_dev::kMaxSweepReqs, round_pairs,
                 round_slots);
  if (ne) {
    ctx->sweep_launches += 1;
    if (ctx->profiling) {
      float ms = 0.0f;
      KREG_CUDA(cudaEventElapsedTime(&ms, S.ev0, S.ev1));
      ctx->sweep_ms += ms;
      if (trace) {
        int n_grad = 0, m_sum = 0;
        for (int e = 0; e < ne; ++e) {
          n_grad += evals[e].grad ? 1 : 0;
          m_sum += evals[e].M;
        }
        std::fprintf(stderr, "kreg-sweep ms=%.4f requests=%d grad=%d m=%d slots=%lld builds=%d\n", ms, ne, n_grad,
                     m_sum, round_slots, nb);
      }
    }
  }
}

void run_round(kreg_ctx* ctx, std::vector<BuildJob>& builds, std::vector<EvalJob>& evals) {
  RoundSlot& S = *round_slot(ctx, 2);
  begin_round(ctx, S, std::move(builds), std::move(evals));
  end_round(ctx, S);
}

double max_point_displacement_dev(kreg_ctx* ctx, const kreg_cloud* Z, const double* built, const double* now) {
  if (Z->n == 0) return 0.0;
  ctx->d_T2.ensure(24);
  ctx->d_disp.ensure(1);
  double T2[24];
  std::memcpy(T2, built, sizeof(double) * 12);
  std::memcpy(T2 + 12, now, sizeof(double) * 12);
  KREG_CUDA(cudaMemcpyAsync(ctx->d_T2.ptr, T2, sizeof(T2), cudaMemcpyHostToDevice, ctx->stream));
  KREG_CUDA(cudaMemsetAsync(ctx->d_disp.ptr, 0, sizeof(unsigned long long), ctx->stream));
  kreg_dev::displacement(Z->x.ptr, Z->y.ptr, Z->z.ptr, Z->n, ctx->d_T2.ptr, ctx->d_disp.ptr, ctx->stream);
  unsigned long long bits = 0;
  KREG_CUDA(cudaMemcpyAsync(&bits, ctx->d_disp.ptr, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream));
  KREG_CUDA(cudaStreamSynchronize(ctx->stream));
  double d2;
  std::memcpy(&d2, &bits, sizeof(d2));
  return std::sqrt(d2);
}

void pairs_export(kreg_ctx* ctx, const kreg_pairs* pc, int64_t* offsets, int32_t* x_index, double* coeff) {
  // reference layout: CSR by ORIGINAL source index j, ascending ORIGINAL i
  kreg_pairs* p = const_cast<kreg_pairs*>(pc);
  const int nz = p->Z ? p->Z->n : 0;
  if (nz && p->slots && !p->index_valid) {
    // builds skip the target indices; the emit is deterministic, so re-run it
    // with write_index set on the unchanged candidate list
    kreg_dev::BuildReq R = p->last_req;
    R.write_index = 1;
    DevBuf<kreg_dev::BuildReq> d;
    d.ensure(1, false, 1.0);
    DevBuf<double> status;
    status.ensure(kreg_dev::kBuildStatus, false, 1.0);
    R.status = status.ptr;
    KREG_CUDA(cudaMemcpyAsync(d.ptr, &R, sizeof(R), cudaMemcpyHostToDevice, ctx->stream));
    kreg_dev::filter_emit_index(d.ptr, nz, ctx->stream);
    KREG_CUDA(cudaGetLastError());
    KREG_CUDA(cudaStreamSynchronize(ctx->stream));
    p->index_valid = true;
  }
  std::vector<int> deg(static_cast<size_t>(nz) + 1, 0), pos(static_cast<size_t>(nz) + 1, 0);
  std::vector<long long> toff(static_cast<size_t>(p->n_tiles) + 1, 0);
  std::vector<int4> sl(static_cast<size_t>(p->slots));
  std::vector<int> si(static_cast<size_t>(p->slots));
  if (nz) {
    KREG_CUDA(cudaMemcpyAsync(deg.data(), p->count.ptr, sizeof(int) * nz, cudaMemcpyDeviceToHost, ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(pos.data(), p->pos.ptr, sizeof(int) * nz, cudaMemcpyDeviceToHost, ctx->stream));
    KREG_CUDA(cudaMemcpyAsync(toff.data(), p->tile_off.ptr, sizeof(long long) * (p->n_tiles + 1),
                              cudaMemcpyDeviceToHost, ctx->stream));
    if (p->slots) {
      KREG_CUDA(cudaMemcpyAsync(sl.data(), p->slot_buf.ptr, sizeof(int4) * p->slots, cudaMemcpyDeviceToHost,
                                ctx->stream));
      KREG_CUDA(cudaMemcpyAsync(si.data(), p->slot_i.ptr, sizeof(int) * p->slots, cudaMemcpyDeviceToHost, ctx->stream));
    }
    KREG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  std::vector<long long> cnt(static_cast<size_t>(nz), 0);
  for (int js = 0; js < nz; ++js) cnt[static_cast<size_t>(p->Z->order[js])] = deg[js];
  offsets[0] = 0;
  for (int j = 0; j < nz; ++j) offsets[j + 1] = offsets[j] + cnt[static_cast<size_t>(j)];
  std::vector<std::pair<int, double>> tmp;
  for (int js = 0; js < nz; ++js) {
    const int j = p->Z->order[js];
    tmp.clear();
    const int ps = pos[static_cast<size_t>(js)];                         // degree-sorted position of js
    const long long tile = toff[static_cast<size_t>(ps >> 5)];             // its tile (sliced ELL)
    for (long long k = 0; k < deg[js]; ++k) {
      const size_t at = static_cast<size_t>(kreg_dev::slot_index(tile, ps & 31, static_cast<int>(k)));
      float lc;
      std::memcpy(&lc, &sl[at].w, sizeof(float));
      tmp.push_back({p->X->order[si[at]], std::exp2(static_cast<double>(lc))});
    }
    std::sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    long long at = offsets[j];
    for (const auto& [i, c] : tmp) {
      x_index[at] = i;
      coeff[at] = c;
      ++at;
    }
  }
}

}  // namespace kreg_host
