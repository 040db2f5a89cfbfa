/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT. See kreg_oracle.h.
 *
 * Plain-C restatement of the reference hot path. Each function cites the
 * reference file:line it follows; evaluation order mirrors the reference
 * (which is compiled with -std=c++20, i.e. no FP contraction) so that, for
 * serial sums, results agree with the compiled reference to the last bit in
 * most cases. Single-threaded by design. */
#include "kreg_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int set_err(int code, const char* msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
  return code;
}

const char* ko_last_error(void) { return g_err; }

/* ------------------------------------------------------------ rng.hpp:11-46 */
uint64_t ko_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t ko_splitmix_derive(uint64_t seed, uint64_t index) {
  uint64_t s = seed ^ (0x9E3779B97F4A7C15ULL * (index + 1));
  return ko_splitmix_next(&s);
}

/* ------------------------------------------------------------ 3x3 helpers */
/* row-major 3x3 */
static void mat_mul(const double* a, const double* b, double* out) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = a[3 * i] * b[j];
      acc += a[3 * i + 1] * b[3 + j];
      acc += a[3 * i + 2] * b[6 + j];
      t[3 * i + j] = acc;
    }
  memcpy(out, t, sizeof(t));
}

static void mat_vec(const double* a, const double* v, double* out) {
  double t[3];
  for (int i = 0; i < 3; ++i) {
    double acc = a[3 * i] * v[0];
    acc += a[3 * i + 1] * v[1];
    acc += a[3 * i + 2] * v[2];
    t[i] = acc;
  }
  memcpy(out, t, sizeof(t));
}

static void iso_rot(const double T[12], double R[9]) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R[3 * r + c] = T[4 * r + c];
}

static void iso_set(double T[12], const double R[9], const double t[3]) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) T[4 * r + c] = R[3 * r + c];
    T[4 * r + 3] = t[r];
  }
}

/* se3.cpp:129-131 apply = R p + t */
static void apply(const double T[12], const double* p, double* out) {
  double R[9], rp[3];
  iso_rot(T, R);
  mat_vec(R, p, rp);
  out[0] = rp[0] + T[3];
  out[1] = rp[1] + T[7];
  out[2] = rp[2] + T[11];
}

/* se3.cpp:147-156 orthonormalized: U V^T of a one-sided Jacobi SVD, det fixed */
static void orthonormalize(const double* Rin, double* out) {
  double w[9], v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  memcpy(w, Rin, sizeof(w));
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < 3; ++i) {
          al += w[3 * i + p] * w[3 * i + p];
          be += w[3 * i + q] * w[3 * i + q];
          ga += w[3 * i + p] * w[3 * i + q];
        }
        if (fabs(ga) <= 1e-300) continue;
        double o = fabs(ga) / sqrt(al * be);
        if (o > off) off = o;
        double zeta = (be - al) / (2.0 * ga);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < 3; ++i) {
          double wp = w[3 * i + p], wq = w[3 * i + q];
          w[3 * i + p] = c * wp - s * wq;
          w[3 * i + q] = s * wp + c * wq;
          double vp = v[3 * i + p], vq = v[3 * i + q];
          v[3 * i + p] = c * vp - s * vq;
          v[3 * i + q] = s * vp + c * vq;
        }
      }
    if (off < 1e-15) break;
  }
  double u[9];
  for (int k = 0; k < 3; ++k) {
    double n = sqrt(w[k] * w[k] + w[3 + k] * w[3 + k] + w[6 + k] * w[6 + k]);
    for (int i = 0; i < 3; ++i) u[3 * i + k] = n > 0 ? w[3 * i + k] / n : 0.0;
  }
  double vt[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) vt[3 * i + j] = v[3 * j + i];
  mat_mul(u, vt, out);
  double det = out[0] * (out[4] * out[8] - out[5] * out[7]) - out[1] * (out[3] * out[8] - out[5] * out[6]) +
               out[2] * (out[3] * out[7] - out[4] * out[6]);
  if (det < 0.0) {
    /* flip the column of the smallest singular value */
    int kmin = 0;
    double smin = 1e300;
    for (int k = 0; k < 3; ++k) {
      double n = sqrt(w[k] * w[k] + w[3 + k] * w[3 + k] + w[6 + k] * w[6 + k]);
      if (n < smin) {
        smin = n;
        kmin = k;
      }
    }
    for (int i = 0; i < 3; ++i) u[3 * i + kmin] = -u[3 * i + kmin];
    mat_mul(u, vt, out);
  }
}

/* se3.cpp:48-76 exp (Rodrigues, half-angle 1-cos, Taylor below 1e-8) */
int ko_se3_exp(const double xi[6], double T[12]) {
  for (int k = 0; k < 6; ++k)
    if (!isfinite(xi[k])) return set_err(KREG_INVALID_ARGUMENT, "exp: twist has non-finite components");
  const double wx = xi[0], wy = xi[1], wz = xi[2];
  const double theta = sqrt(wx * wx + wy * wy + wz * wz);
  const double W[9] = {0.0, -wz, wy, wz, 0.0, -wx, -wy, wx, 0.0};
  double W2[9];
  mat_mul(W, W, W2);
  double R[9], V[9];
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (theta < 1e-8) {
    for (int k = 0; k < 9; ++k) {
      R[k] = (I[k] + W[k]) + 0.5 * W2[k];
      V[k] = (I[k] + 0.5 * W[k]) + W2[k] / 6.0;
    }
  } else {
    const double t2 = theta * theta;
    const double s = sin(theta);
    const double hs = sin(0.5 * theta);
    const double omc = 2.0 * hs * hs;
    const double a = s / theta;
    const double b = omc / t2;
    const double c = (theta - s) / (t2 * theta);
    for (int k = 0; k < 9; ++k) {
      R[k] = (I[k] + a * W[k]) + b * W2[k];
      V[k] = (I[k] + b * W[k]) + c * W2[k];
    }
  }
  double t[3];
  mat_vec(V, xi + 3, t);
  iso_set(T, R, t);
  return 0;
}

/* se3.cpp:109-120 compose */
void ko_se3_compose(const double a[12], const double b[12], double out[12]) {
  double Ra[9], Rb[9], R[9], t[3];
  iso_rot(a, Ra);
  iso_rot(b, Rb);
  mat_mul(Ra, Rb, R);
  const double tb[3] = {b[3], b[7], b[11]};
  mat_vec(Ra, tb, t);
  t[0] = t[0] + a[3];
  t[1] = t[1] + a[7];
  t[2] = t[2] + a[11];
  /* Gram drift check (Frobenius) */
  double g[9], Rt[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rt[3 * i + j] = R[3 * j + i];
  mat_mul(Rt, R, g);
  double fro = 0.0;
  for (int k = 0; k < 9; ++k) {
    const double d = g[k] - ((k % 4 == 0) ? 1.0 : 0.0);
    fro += d * d;
  }
  if (sqrt(fro) > 1e-7) orthonormalize(R, R);
  iso_set(out, R, t);
}

/* se3.cpp:122-127 inverse */
void ko_se3_inverse(const double T[12], double out[12]) {
  double R[9], Rt[9], t[3];
  iso_rot(T, R);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rt[3 * i + j] = R[3 * j + i];
  const double tt[3] = {T[3], T[7], T[11]};
  mat_vec(Rt, tt, t);
  t[0] = -t[0];
  t[1] = -t[1];
  t[2] = -t[2];
  iso_set(out, Rt, t);
}

/* --------------------------------------------------------- kernel math */
/* kernels.hpp:37-42 */
static double sqdist(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

/* kernels.hpp:45-47 */
static double kernel_sq(double sq, double sigma, double l) {
  return sigma * sigma * exp(-sq / (2.0 * l * l));
}

/* kernels.cpp:18-53 */
double ko_feature_coefficient(const double* u, const double* v, const kreg_cloud_view* schema,
                              const kreg_kernel_params* params) {
  if (schema->n_channels == 0) return 1.0;
  double c = 1.0;
  int off = 0;
  for (int k = 0; k < schema->n_channels; ++k) {
    const int dim = schema->channels[k].dim;
    const kreg_channel_params* cp = &params->per_channel[k];
    if (cp->form == KREG_FORM_LINEAR) {
      double dot = 0.0;
      for (int d = 0; d < dim; ++d) dot += u[off + d] * v[off + d];
      c *= dot;
    } else {
      double sq = 0.0;
      for (int d = 0; d < dim; ++d) {
        const double diff = u[off + d] - v[off + d];
        sq += diff * diff;
      }
      c *= kernel_sq(sq, cp->sigma, cp->lengthscale);
    }
    off += dim;
  }
  return c;
}

/* kernels.cpp:70-95 check_kernel_params (message subset) */
static int check_params(const kreg_kernel_params* p, const kreg_cloud_view* schema) {
  if (!(p->lengthscale > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "kernel params: geometric lengthscale must be > 0");
  if (!(p->sigma > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "kernel params: sigma must be > 0");
  if (p->n_channels != schema->n_channels) return set_err(KREG_INVALID_ARGUMENT, "kernel params: channel entries do not match schema");
  for (int k = 0; k < p->n_channels; ++k) {
    if (p->per_channel[k].form == KREG_FORM_SQUARED_EXPONENTIAL && !(p->per_channel[k].lengthscale > 0.0))
      return set_err(KREG_INVALID_ARGUMENT, "kernel params: channel lengthscale must be > 0");
    if (!(p->per_channel[k].sigma > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "kernel params: channel sigma must be > 0");
  }
  return 0;
}

static int same_schema(const kreg_cloud_view* X, const kreg_cloud_view* Z) {
  if (X->n_channels != Z->n_channels) return 0;
  for (int k = 0; k < X->n_channels; ++k) {
    if (X->channels[k].dim != Z->channels[k].dim || X->channels[k].kind != Z->channels[k].kind) return 0;
    if (strcmp(X->channels[k].name, Z->channels[k].name) != 0) return 0;
  }
  return 1;
}

/* ------------------------------------------------------- pair list (A6) */
struct ko_pairs {
  int64_t* offsets;
  int32_t* x_index;
  double* coeff;
  int64_t n;
  int32_t n_x, n_z;
  double built_at_lengthscale, cutoff_radius, c_min;
  double build_transform[12];
};

void ko_pairs_destroy(ko_pairs* p) {
  if (!p) return;
  free(p->offsets);
  free(p->x_index);
  free(p->coeff);
  free(p);
}

void ko_pairs_export(const ko_pairs* p, int64_t* offsets, int32_t* x_index, double* coeff) {
  memcpy(offsets, p->offsets, sizeof(int64_t) * (size_t)(p->n_z + 1));
  if (p->n) {
    memcpy(x_index, p->x_index, sizeof(int32_t) * (size_t)p->n);
    memcpy(coeff, p->coeff, sizeof(double) * (size_t)p->n);
  }
}

/* hash_grid.hpp:41-50 cell coordinates; the grid here is a sorted key list
 * (same candidate set as the reference's unordered_map CSR; the final per-j
 * hit order is by i either way, inner_product.cpp:77-78). */
typedef struct {
  uint64_t key;
  int32_t i;
} keyed;

static int cmp_keyed(const void* a, const void* b) {
  const keyed* x = (const keyed*)a;
  const keyed* y = (const keyed*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->i - y->i;
}

static uint64_t cell_key(int64_t x, int64_t y, int64_t z) {
  const uint64_t bias = 1u << 20;
  return (((uint64_t)(x + (int64_t)bias) & 0x1FFFFF) << 42) | (((uint64_t)(y + (int64_t)bias) & 0x1FFFFF) << 21) |
         ((uint64_t)(z + (int64_t)bias) & 0x1FFFFF);
}

static int cmp_hit(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* inner_product.cpp:37-95 build_pairs ; reference.cpp:9-37 dense_pairs */
int ko_build_pairs(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double T[12],
                   const kreg_kernel_params* params, double cutoff_multiplier, double c_min,
                   int dense, ko_pairs** out, int64_t* n_pairs) {
  if (!same_schema(X, Z)) return set_err(KREG_INVALID_ARGUMENT, "schema mismatch");
  int rc = check_params(params, X);
  if (rc) return rc;
  if (!(cutoff_multiplier >= 1.0)) return set_err(KREG_INVALID_ARGUMENT, "build_pairs: cutoff_multiplier must be >= 1");
  if (c_min < 0.0 || c_min >= 1.0) return set_err(KREG_INVALID_ARGUMENT, "build_pairs: c_min must lie in [0, 1)");

  ko_pairs* p = (ko_pairs*)calloc(1, sizeof(ko_pairs));
  p->built_at_lengthscale = params->lengthscale;
  p->cutoff_radius = cutoff_multiplier * params->lengthscale;
  p->c_min = c_min;
  memcpy(p->build_transform, T, sizeof(double) * 12);
  p->n_x = X->n;
  p->n_z = Z->n;
  p->offsets = (int64_t*)calloc((size_t)Z->n + 1, sizeof(int64_t));
  *out = p;
  *n_pairs = 0;
  if (X->n == 0 || Z->n == 0) return 0;

  const double cutoff_sq = p->cutoff_radius * p->cutoff_radius;
  const int geo = X->n_channels == 0;
  const int dim = X->dim;

  /* hash_grid.cpp:8-36: origin = componentwise min, cell = cutoff */
  double origin[3] = {X->xyz[0], X->xyz[1], X->xyz[2]};
  for (int i = 0; i < X->n; ++i)
    for (int k = 0; k < 3; ++k)
      if (X->xyz[3 * i + k] < origin[k]) origin[k] = X->xyz[3 * i + k];
  const double inv_cell = 1.0 / p->cutoff_radius;
  keyed* grid = NULL;
  if (!dense) {
    grid = (keyed*)malloc(sizeof(keyed) * (size_t)X->n);
    for (int i = 0; i < X->n; ++i) {
      const double* x = X->xyz + 3 * i;
      grid[i].key = cell_key((int64_t)floor((x[0] - origin[0]) * inv_cell), (int64_t)floor((x[1] - origin[1]) * inv_cell),
                             (int64_t)floor((x[2] - origin[2]) * inv_cell));
      grid[i].i = i;
    }
    qsort(grid, (size_t)X->n, sizeof(keyed), cmp_keyed);
  }

  int64_t cap = 1024, n = 0;
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  double* cf = (double*)malloc(sizeof(double) * (size_t)cap);
  int32_t* hits = (int32_t*)malloc(sizeof(int32_t) * (size_t)X->n);
  for (int j = 0; j < Z->n; ++j) {
    double q[3];
    apply(T, Z->xyz + 3 * j, q);
    int nh = 0;
    if (dense) {
      for (int i = 0; i < X->n; ++i) hits[nh++] = i;
    } else {
      const int64_t cx = (int64_t)floor((q[0] - origin[0]) * inv_cell);
      const int64_t cy = (int64_t)floor((q[1] - origin[1]) * inv_cell);
      const int64_t cz = (int64_t)floor((q[2] - origin[2]) * inv_cell);
      for (int64_t dz = -1; dz <= 1; ++dz)
        for (int64_t dy = -1; dy <= 1; ++dy)
          for (int64_t dx = -1; dx <= 1; ++dx) {
            const uint64_t key = cell_key(cx + dx, cy + dy, cz + dz);
            /* lower bound */
            int64_t lo = 0, hi = X->n;
            while (lo < hi) {
              const int64_t mid = (lo + hi) / 2;
              if (grid[mid].key < key) lo = mid + 1;
              else hi = mid;
            }
            for (int64_t s = lo; s < X->n && grid[s].key == key; ++s) hits[nh++] = grid[s].i;
          }
      qsort(hits, (size_t)nh, sizeof(int32_t), cmp_hit);
    }
    for (int h = 0; h < nh; ++h) {
      const int i = hits[h];
      if (sqdist(X->xyz + 3 * i, q) > cutoff_sq) continue;
      double c = 1.0;
      if (!geo) {
        c = ko_feature_coefficient(X->features + (size_t)i * dim, Z->features + (size_t)j * dim, X, params);
        if (!(c > c_min)) continue;
      }
      if (n == cap) {
        cap *= 2;
        idx = (int32_t*)realloc(idx, sizeof(int32_t) * (size_t)cap);
        cf = (double*)realloc(cf, sizeof(double) * (size_t)cap);
      }
      idx[n] = i;
      cf[n] = c;
      ++n;
    }
    p->offsets[j + 1] = n;
  }
  free(hits);
  free(grid);
  p->x_index = idx;
  p->coeff = cf;
  p->n = n;
  *n_pairs = n;
  return 0;
}

/* reduce.hpp:12-23 pairwise_sum over stride-`w` records of doubles */
static void pairwise_sum(const double* xs, size_t n, int w, double* out) {
  if (n == 0) {
    for (int k = 0; k < w; ++k) out[k] = 0.0;
    return;
  }
  if (n <= 8) {
    for (int k = 0; k < w; ++k) out[k] = xs[k];
    for (size_t i = 1; i < n; ++i)
      for (int k = 0; k < w; ++k) out[k] = out[k] + xs[i * (size_t)w + (size_t)k];
    return;
  }
  const size_t half = n / 2;
  double a[8], b[8];
  pairwise_sum(xs, half, w, a);
  pairwise_sum(xs + half * (size_t)w, n - half, w, b);
  for (int k = 0; k < w; ++k) out[k] = a[k] + b[k];
}

/* inner_product.cpp:97-119 */
double ko_inner_product(const ko_pairs* p, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                        const double T[12], const kreg_kernel_params* params) {
  if (p->n == 0) return 0.0;
  double* partial = (double*)calloc((size_t)p->n_z, sizeof(double));
  /* per-j partials, fixed-shape reduction: thread-count independent (reduce.hpp:8-11) */
#pragma omp parallel for schedule(dynamic, 64)
  for (int j = 0; j < p->n_z; ++j) {
    double q[3];
    apply(T, Z->xyz + 3 * j, q);
    double acc = 0.0;
    for (int64_t e = p->offsets[j]; e < p->offsets[j + 1]; ++e) {
      const int i = p->x_index[e];
      acc += p->coeff[e] * kernel_sq(sqdist(X->xyz + 3 * i, q), params->sigma, params->lengthscale);
    }
    partial[j] = acc;
  }
  double total;
  pairwise_sum(partial, (size_t)p->n_z, 1, &total);
  free(partial);
  return total;
}

/* inner_product.cpp:121-152 ; FGradPartial = {f, gv[3], gw[3]} (:16-24) */
void ko_objective_and_gradient(const ko_pairs* p, const kreg_cloud_view* X,
                               const kreg_cloud_view* Z, const double T[12],
                               const kreg_kernel_params* params, double out[7]) {
  for (int k = 0; k < 7; ++k) out[k] = 0.0;
  if (p->n == 0) return;
  const double inv_l2 = 1.0 / (params->lengthscale * params->lengthscale);
  double* partial = (double*)calloc((size_t)p->n_z * 7, sizeof(double));
#pragma omp parallel for schedule(dynamic, 64)
  for (int j = 0; j < p->n_z; ++j) {
    double q[3];
    apply(T, Z->xyz + 3 * j, q);
    double* a = partial + 7 * (size_t)j;
    for (int64_t e = p->offsets[j]; e < p->offsets[j + 1]; ++e) {
      const double* x = X->xyz + 3 * p->x_index[e];
      const double k = kernel_sq(sqdist(x, q), params->sigma, params->lengthscale);
      const double w = p->coeff[e] * k;
      a[0] += w;
      a[1] += w * (x[0] - q[0]);
      a[2] += w * (x[1] - q[1]);
      a[3] += w * (x[2] - q[2]);
      const double cx = q[1] * x[2] - q[2] * x[1];
      const double cy = q[2] * x[0] - q[0] * x[2];
      const double cz = q[0] * x[1] - q[1] * x[0];
      a[4] += w * cx;
      a[5] += w * cy;
      a[6] += w * cz;
    }
  }
  double tot[7];
  pairwise_sum(partial, (size_t)p->n_z, 7, tot);
  free(partial);
  out[0] = tot[0];
  for (int k = 0; k < 3; ++k) {
    out[1 + k] = tot[4 + k] * inv_l2; /* omega */
    out[4 + k] = tot[1 + k] * inv_l2; /* v */
  }
}

/* Second-order step-size terms along xi (north_star item (4); diagnostic
 * only, the reference has no second-order step: SURVEY.md §8 A15).
 * F(eps) = sum c k(|x_i - q_j(eps)|^2) with q_j(eps) = exp(eps xi) T z_j
 * (left perturbation, registration.cpp:69), so q' = u = omega x q + v and
 * q'' = omega x u at eps = 0; with d = x - q:
 *   F'  = sum w (d.u) / l^2
 *   F'' = sum w [ (d.u)^2 / l^4 - (|u|^2 - d.(omega x u)) / l^2 ]
 * out = {F, F'(0), F''(0)}. */
void ko_directional_terms(const ko_pairs* p, const kreg_cloud_view* X, const kreg_cloud_view* Z,
                          const double T[12], const double xi[6], const kreg_kernel_params* params, double out[3]) {
  out[0] = out[1] = out[2] = 0.0;
  if (p->n == 0) return;
  const double inv_l2 = 1.0 / (params->lengthscale * params->lengthscale);
  double* partial = (double*)calloc((size_t)p->n_z * 3, sizeof(double));
#pragma omp parallel for schedule(dynamic, 64)
  for (int j = 0; j < p->n_z; ++j) {
    double q[3];
    apply(T, Z->xyz + 3 * j, q);
    const double* w_ = xi;
    const double u[3] = {w_[1] * q[2] - w_[2] * q[1] + xi[3], w_[2] * q[0] - w_[0] * q[2] + xi[4],
                         w_[0] * q[1] - w_[1] * q[0] + xi[5]};
    const double ou[3] = {w_[1] * u[2] - w_[2] * u[1], w_[2] * u[0] - w_[0] * u[2], w_[0] * u[1] - w_[1] * u[0]};
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    double* a = partial + 3 * (size_t)j;
    for (int64_t e = p->offsets[j]; e < p->offsets[j + 1]; ++e) {
      const double* x = X->xyz + 3 * p->x_index[e];
      const double w = p->coeff[e] * kernel_sq(sqdist(x, q), params->sigma, params->lengthscale);
      const double d[3] = {x[0] - q[0], x[1] - q[1], x[2] - q[2]};
      const double du = d[0] * u[0] + d[1] * u[1] + d[2] * u[2];
      const double dou = d[0] * ou[0] + d[1] * ou[1] + d[2] * ou[2];
      a[0] += w;
      a[1] += w * du * inv_l2;
      a[2] += w * (du * du * inv_l2 * inv_l2 - (uu - dou) * inv_l2);
    }
  }
  pairwise_sum(partial, (size_t)p->n_z, 3, out);
  free(partial);
}

/* inner_product.cpp:238-246 */
double ko_max_point_displacement(const kreg_cloud_view* Z, const double built[12], const double now[12]) {
  double worst = 0.0;
  for (int j = 0; j < Z->n; ++j) {
    double a[3], b[3];
    apply(now, Z->xyz + 3 * j, a);
    apply(built, Z->xyz + 3 * j, b);
    const double d = sqdist(a, b);
    if (d > worst) worst = d;
  }
  return sqrt(worst);
}

/* point_cloud.cpp:69-87 */
double ko_diameter(const kreg_cloud_view* X) {
  const int n = X->n;
  if (n <= 1) return 0.0;
  if (n <= 2000) {
    double best = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        const double d = sqdist(X->xyz + 3 * i, X->xyz + 3 * j);
        if (d > best) best = d;
      }
    return sqrt(best);
  }
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) lo[k] = hi[k] = X->xyz[k];
  for (int i = 1; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      const double v = X->xyz[3 * i + k];
      if (v < lo[k]) lo[k] = v;
      if (v > hi[k]) hi[k] = v;
    }
  const double d[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  return sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
}

/* registration.cpp:36-52 */
double ko_anneal_step(double lengthscale, const double* history, int n, const kreg_registration_config* c) {
  const int window = c->stabilization_window;
  if (n < window) return lengthscale;
  const double* last = history + (n - window);
  double lo = last[0], hi = last[0], scale = fabs(last[0]);
  for (int k = 0; k < window; ++k) {
    lo = fmin(lo, last[k]);
    hi = fmax(hi, last[k]);
    scale = fmax(scale, fabs(last[k]));
  }
  if (hi - lo > c->stabilization_rel_tol * fmax(scale, DBL_MIN)) return lengthscale;
  const double decayed = lengthscale * c->decay_factor;
  return decayed >= c->min_lengthscale ? decayed : lengthscale;
}

/* registration.cpp:12-34 */
int ko_check_config(const kreg_registration_config* c) {
  if (!(c->decay_factor > 0.0 && c->decay_factor < 1.0)) return set_err(KREG_INVALID_ARGUMENT, "config: decay_factor must lie in (0, 1)");
  if (!(c->min_lengthscale > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "config: min_lengthscale must be > 0");
  if (!(c->min_lengthscale <= c->init_lengthscale)) return set_err(KREG_INVALID_ARGUMENT, "config: min_lengthscale must not exceed init_lengthscale");
  if (!(c->subsequent_lengthscale > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "config: subsequent_lengthscale must be > 0");
  if (c->max_iterations < 1) return set_err(KREG_INVALID_ARGUMENT, "config: max_iterations must be >= 1");
  if (c->stabilization_window < 1) return set_err(KREG_INVALID_ARGUMENT, "config: stabilization_window must be >= 1");
  if (!(c->stabilization_rel_tol > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "config: stabilization_rel_tol must be > 0");
  if (!(c->step_init > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "config: step_init must be > 0");
  if (!(c->step_shrink > 0.0 && c->step_shrink < 1.0)) return set_err(KREG_INVALID_ARGUMENT, "config: step_shrink must lie in (0, 1)");
  if (!(c->step_grow >= 1.0)) return set_err(KREG_INVALID_ARGUMENT, "config: step_grow must be >= 1");
  if (c->max_backtracks < 0) return set_err(KREG_INVALID_ARGUMENT, "config: max_backtracks must be >= 0");
  if (!(c->convergence_twist_norm > 0.0)) return set_err(KREG_INVALID_ARGUMENT, "config: convergence_twist_norm must be > 0");
  if (!(c->cutoff_multiplier >= 1.0)) return set_err(KREG_INVALID_ARGUMENT, "config: cutoff_multiplier must be >= 1");
  if (c->c_min < 0.0 || c->c_min >= 1.0) return set_err(KREG_INVALID_ARGUMENT, "config: c_min must lie in [0, 1)");
  return 0;
}

static void push_trace(kreg_registration_result* r, int it, double f, double ind, double l, double step,
                       double tn, int64_t pc, int rebuilt) {
  if (it >= r->trace_capacity) return;
  if (r->objective_trace) r->objective_trace[it] = f;
  if (r->indicator_trace) r->indicator_trace[it] = ind;
  if (r->lengthscale_trace) r->lengthscale_trace[it] = l;
  if (r->step_trace) r->step_trace[it] = step;
  if (r->twist_norm_trace) r->twist_norm_trace[it] = tn;
  if (r->pair_count_trace) r->pair_count_trace[it] = pc;
  if (r->rebuild_trace) r->rebuild_trace[it] = (uint8_t)rebuilt;
}

/* Replay log (parity tests): per iteration, the transform T the iteration
 * evaluates and the build transform / lengthscale of the pair list it uses
 * (after the rebuild rule, registration.cpp:123-130). */
static double* g_log_T = NULL;
static double* g_log_Tb = NULL;
static double* g_log_l = NULL;
static int g_log_cap = 0;
void ko_set_iteration_log(double* T, double* Tb, double* l, int cap) {
  g_log_T = T;
  g_log_Tb = Tb;
  g_log_l = l;
  g_log_cap = cap;
}

/* registration.cpp:100-189 register_clouds */
int ko_register_clouds(const kreg_cloud_view* X, const kreg_cloud_view* Z, const double initial[12],
                       const kreg_kernel_params* params, const kreg_registration_config* cfg,
                       kreg_registration_result* res) {
  int rc = ko_check_config(cfg);
  if (rc) return rc;
  if (!same_schema(X, Z)) return set_err(KREG_INVALID_ARGUMENT, "register: schema mismatch");

  const double diam = ko_diameter(X);
  const double v_scale = diam > 0.0 ? diam : 1.0;
  const double denom = sqrt((double)(X->n > 1 ? X->n : 1) * (double)(Z->n > 1 ? Z->n : 1));

  double lengthscale = cfg->init_lengthscale;
  kreg_kernel_params wp = *params;
  wp.lengthscale = lengthscale;
  double T[12];
  memcpy(T, initial, sizeof(T));
  ko_pairs* pairs = NULL;
  int64_t np = 0;
  rc = ko_build_pairs(X, Z, T, &wp, cfg->cutoff_multiplier, cfg->c_min, 0, &pairs, &np);
  if (rc) return rc;
  if (np == 0) {
    char msg[128];
    snprintf(msg, sizeof(msg), "no overlapping pairs within cutoff radius %f m", pairs->cutoff_radius);
    ko_pairs_destroy(pairs);
    return set_err(KREG_NO_OVERLAP, msg);
  }

  double* window = (double*)malloc(sizeof(double) * (size_t)cfg->max_iterations);
  int nwin = 0;
  double step_factor = 1.0;
  int it_count = 0;
  double last_ind = 0.0;
  res->converged = 0;

  for (int iter = 0; iter < cfg->max_iterations; ++iter) {
    int rebuilt = 0;
    if (pairs->built_at_lengthscale != lengthscale ||
        ko_max_point_displacement(Z, pairs->build_transform, T) > 0.5 * pairs->cutoff_radius) {
      double Tb[12];
      memcpy(Tb, T, sizeof(Tb));
      ko_pairs_destroy(pairs);
      ko_build_pairs(X, Z, Tb, &wp, cfg->cutoff_multiplier, cfg->c_min, 0, &pairs, &np);
      rebuilt = 1;
      if (np == 0) break;
    }

    if (iter < g_log_cap) {
      if (g_log_T) memcpy(g_log_T + 12 * (size_t)iter, T, sizeof(double) * 12);
      if (g_log_Tb) memcpy(g_log_Tb + 12 * (size_t)iter, pairs->build_transform, sizeof(double) * 12);
      if (g_log_l) g_log_l[iter] = lengthscale;
    }
    double ev[7];
    ko_objective_and_gradient(pairs, X, Z, T, &wp, ev);
    const double gnorm = sqrt((ev[1] * ev[1] + ev[2] * ev[2] + ev[3] * ev[3]) + (ev[4] * ev[4] + ev[5] * ev[5] + ev[6] * ev[6]));
    const double step0 = cfg->step_init * lengthscale * step_factor;

    double accepted_step = 0.0, f_now = ev[0], twist_norm = 0.0;
    if (gnorm > 0.0 && step0 * gnorm > 1e-12 * fmax(fabs(ev[0]), 1.0)) {
      double dir[6];
      const double s = 1.0 / gnorm;
      for (int k = 0; k < 6; ++k) dir[k] = ev[1 + k] * s;
      /* registration.cpp:63-75 backtracking_search */
      double eps = step0;
      int accepted = 0, backtracks = 0;
      double fval = ev[0], cand[12];
      for (int k = 0; k <= cfg->max_backtracks; ++k) {
        double tw[6], E[12];
        for (int m = 0; m < 6; ++m) tw[m] = dir[m] * eps;
        ko_se3_exp(tw, E);
        ko_se3_compose(E, T, cand);
        const double f = ko_inner_product(pairs, X, Z, cand, &wp);
        if (f > ev[0]) {
          accepted = 1;
          backtracks = k;
          fval = f;
          break;
        }
        eps *= cfg->step_shrink;
      }
      if (accepted) {
        accepted_step = eps;
        f_now = fval;
        double applied[6], E[12], Tn[12];
        for (int m = 0; m < 6; ++m) applied[m] = dir[m] * accepted_step;
        ko_se3_exp(applied, E);
        ko_se3_compose(E, T, Tn);
        memcpy(T, Tn, sizeof(T));
        twist_norm = sqrt(applied[0] * applied[0] + applied[1] * applied[1] + applied[2] * applied[2]) +
                     sqrt(applied[3] * applied[3] + applied[4] * applied[4] + applied[5] * applied[5]) / v_scale;
        step_factor = backtracks == 0 ? fmin(step_factor * cfg->step_grow, 1e3)
                                      : fmax(step_factor * pow(cfg->step_shrink, backtracks), 1e-6);
      } else {
        step_factor = fmax(step_factor * cfg->step_shrink, 1e-6);
      }
    }

    const double ind = f_now / denom;
    push_trace(res, it_count, f_now, ind, lengthscale, accepted_step, twist_norm, np, rebuilt);
    ++it_count;
    last_ind = ind;
    window[nwin++] = ind;

    const int at_floor = lengthscale * cfg->decay_factor < cfg->min_lengthscale;
    if (at_floor && twist_norm < cfg->convergence_twist_norm) {
      res->converged = 1;
      break;
    }
    const double next = ko_anneal_step(lengthscale, window, nwin, cfg);
    if (next != lengthscale) {
      lengthscale = next;
      wp.lengthscale = lengthscale;
      nwin = 0;
      step_factor = 1.0;
    }
  }
  ko_pairs_destroy(pairs);
  free(window);
  memcpy(res->transform, T, sizeof(T));
  res->iterations = it_count;
  res->final_indicator = it_count ? last_ind : 0.0;
  res->sweeps = 0;
  res->rebuilds = 0;
  return 0;
}


/* ------------------------------------------------------------ frame ingest
 * Plain restatement of image.cpp:144-155, selector.cpp:21-125 and
 * projection.cpp:30-75 (the detector is re-run every threshold round, as the
 * reference does). */
void ko_to_gray(const uint8_t* rgb, int channels, int w, int h, uint8_t* gray) {
  for (long i = 0; i < (long)w * h; ++i) {
    if (channels == 1) {
      gray[i] = rgb[i];
    } else {
      const uint8_t* p = rgb + i * channels;
      gray[i] = (uint8_t)((299 * p[0] + 587 * p[1] + 114 * p[2]) / 1000);
    }
  }
}

static const int ko_circle[16][2] = {
    {0, -3}, {1, -3}, {2, -2}, {3, -1}, {3, 0},  {3, 1},  {2, 2},  {1, 3},
    {0, 3},  {-1, 3}, {-2, 2}, {-3, 1}, {-3, 0}, {-3, -1}, {-2, -2}, {-1, -3},
};

int ko_is_corner(const uint8_t* gray, int w, int u, int v, double t) {
  const double center = gray[(long)v * w + u];
  int state[16];
  for (int s = 0; s < 16; ++s) {
    const double p = gray[(long)(v + ko_circle[s][1]) * w + u + ko_circle[s][0]];
    state[s] = p > center + t ? 1 : (p < center - t ? -1 : 0);
  }
  for (int want = 1; want >= -1; want -= 2) {
    int run = 0;
    for (int s = 0; s < 32; ++s) {
      if (state[s & 15] == want) {
        if (++run >= 9) return 1;
      } else {
        run = 0;
      }
    }
  }
  return 0;
}

long ko_select_points(const uint8_t* rgb, int channels, int w, int h, const uint8_t* valid,
                      const kreg_selector_config* sel, int32_t* pixels, double* threshold, int* in_band,
                      int* fallback) {
  uint8_t* gray = (uint8_t*)malloc((size_t)w * h + 1);
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * 2 * ((size_t)w * h + 1));
  ko_to_gray(rgb, channels, w, h, gray);
  double t = sel->initial_threshold;
  long best_gap = -1, best_n = 0;
  *threshold = 0.0;
  *in_band = 0;
  *fallback = 0;
  int done = 0;
  for (int round = 0; round < sel->max_adjust_rounds && !done; ++round) {
    long n = 0;
    for (int v = 3; v < h - 3; ++v)
      for (int u = 3; u < w - 3; ++u)
        if (ko_is_corner(gray, w, u, v, t) && valid[(long)v * w + u]) {
          cur[2 * n] = u;
          cur[2 * n + 1] = v;
          ++n;
        }
    const long gap = n < sel->target_min ? sel->target_min - n : n > sel->target_max ? n - sel->target_max : 0;
    if (best_gap < 0 || gap < best_gap) {
      best_gap = gap;
      best_n = n;
      *threshold = t;
      memcpy(pixels, cur, sizeof(int32_t) * 2 * (size_t)n);
    }
    if (gap == 0) {
      *in_band = 1;
      done = 1;
      break;
    }
    if (n > sel->target_max) {
      t *= sel->adjust_factor;
    } else {
      if (t <= 0.5) break;
      t = t / sel->adjust_factor > 0.5 ? t / sel->adjust_factor : 0.5;
    }
  }
  if (!*in_band && best_n < sel->target_min) {
    best_n = 0;
    for (int v = 0; v < h; ++v)
      for (int u = 0; u < w; ++u)
        if (valid[(long)v * w + u]) {
          pixels[2 * best_n] = u;
          pixels[2 * best_n + 1] = v;
          ++best_n;
        }
    *fallback = 1;
  }
  free(gray);
  free(cur);
  return best_n;
}

long ko_depth_rgb_to_cloud(const uint16_t* depth, const uint8_t* rgb, int channels, const float* sem, int sem_ch,
                           int w, int h, const kreg_camera_intrinsics* in, const kreg_selector_config* sel,
                           double* xyz, double* feat, int* fallback, int* in_band) {
  uint8_t* valid = (uint8_t*)calloc((size_t)w * h + 1, 1);
  int32_t* px = (int32_t*)malloc(sizeof(int32_t) * 2 * ((size_t)w * h + 1));
  for (int v = in->skip_top_rows; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const uint16_t d = depth[(long)v * w + u];
      if (d == 0) continue;
      if (d * in->depth_scale > in->max_depth) continue;
      valid[(long)v * w + u] = 1;
    }
  double thr;
  const long n = ko_select_points(rgb, channels, w, h, valid, sel, px, &thr, in_band, fallback);
  const int D = 3 + (sem ? sem_ch : 0);
  for (long k = 0; k < n; ++k) {
    const int u = px[2 * k], v = px[2 * k + 1];
    const long i = (long)v * w + u;
    const double dm = depth[i] * in->depth_scale;
    xyz[3 * k] = dm * ((u - in->cx) / in->fx);
    xyz[3 * k + 1] = dm * ((v - in->cy) / in->fy);
    xyz[3 * k + 2] = dm * 1.0;
    const long end = (long)w * h * channels;
    for (int c = 0; c < 3; ++c) {
      const long at = i * channels + c;
      feat[D * k + c] = (at < end ? rgb[at] : 0) / 255.0;
    }
    for (int c = 0; sem && c < sem_ch; ++c) feat[D * k + 3 + c] = sem[i * sem_ch + c];
  }
  free(valid);
  free(px);
  return n;
}
