// Host SE(3) math of the registration loop (row-major 3x4 isometries).
// Same formulas and evaluation order as the reference (se3.cpp:15-156) so the
// transform updates of the host loop match it to the last bit in FP64.
#pragma once

#include <cmath>
#include <cstring>

namespace kreg_se3 {

inline void mat_mul(const double* a, const double* b, double* out) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = a[3 * i] * b[j];
      acc += a[3 * i + 1] * b[3 + j];
      acc += a[3 * i + 2] * b[6 + j];
      t[3 * i + j] = acc;
    }
  std::memcpy(out, t, sizeof(t));
}

inline void mat_vec(const double* a, const double* v, double* out) {
  double t[3];
  for (int i = 0; i < 3; ++i) {
    double acc = a[3 * i] * v[0];
    acc += a[3 * i + 1] * v[1];
    acc += a[3 * i + 2] * v[2];
    t[i] = acc;
  }
  std::memcpy(out, t, sizeof(t));
}

inline void rot_of(const double* T, double* R) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R[3 * r + c] = T[4 * r + c];
}

inline void set_iso(double* T, const double* R, const double* t) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) T[4 * r + c] = R[3 * r + c];
    T[4 * r + 3] = t[r];
  }
}

inline void identity(double* T) {
  static const double I[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
  std::memcpy(T, I, sizeof(I));
}

// se3.cpp:147-156: nearest rotation (U V^T of a one-sided Jacobi SVD).
inline void orthonormalize(const double* Rin, double* out) {
  double w[9], v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  std::memcpy(w, Rin, sizeof(w));
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
        if (std::fabs(ga) <= 1e-300) continue;
        off = std::fmax(off, std::fabs(ga) / std::sqrt(al * be));
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < 3; ++i) {
          const double wp = w[3 * i + p], wq = w[3 * i + q];
          w[3 * i + p] = c * wp - s * wq;
          w[3 * i + q] = s * wp + c * wq;
          const double vp = v[3 * i + p], vq = v[3 * i + q];
          v[3 * i + p] = c * vp - s * vq;
          v[3 * i + q] = s * vp + c * vq;
        }
      }
    if (off < 1e-15) break;
  }
  double u[9], sv[3];
  for (int k = 0; k < 3; ++k) {
    sv[k] = std::sqrt(w[k] * w[k] + w[3 + k] * w[3 + k] + w[6 + k] * w[6 + k]);
    for (int i = 0; i < 3; ++i) u[3 * i + k] = sv[k] > 0 ? w[3 * i + k] / sv[k] : 0.0;
  }
  double vt[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) vt[3 * i + j] = v[3 * j + i];
  mat_mul(u, vt, out);
  const double det = out[0] * (out[4] * out[8] - out[5] * out[7]) - out[1] * (out[3] * out[8] - out[5] * out[6]) +
                     out[2] * (out[3] * out[7] - out[4] * out[6]);
  if (det < 0.0) {
    int kmin = 0;
    for (int k = 1; k < 3; ++k)
      if (sv[k] < sv[kmin]) kmin = k;
    for (int i = 0; i < 3; ++i) u[3 * i + kmin] = -u[3 * i + kmin];
    mat_mul(u, vt, out);
  }
}

// se3.cpp:48-76. Returns false on non-finite input.
inline bool exp(const double* xi, double* T) {
  for (int k = 0; k < 6; ++k)
    if (!std::isfinite(xi[k])) return false;
  const double wx = xi[0], wy = xi[1], wz = xi[2];
  const double theta = std::sqrt(wx * wx + wy * wy + wz * wz);
  const double W[9] = {0.0, -wz, wy, wz, 0.0, -wx, -wy, wx, 0.0};
  double W2[9];
  mat_mul(W, W, W2);
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double R[9], V[9];
  if (theta < 1e-8) {
    for (int k = 0; k < 9; ++k) {
      R[k] = (I[k] + W[k]) + 0.5 * W2[k];
      V[k] = (I[k] + 0.5 * W[k]) + W2[k] / 6.0;
    }
  } else {
    const double t2 = theta * theta;
    const double s = std::sin(theta);
    const double hs = std::sin(0.5 * theta);
    const double omc = 2.0 * hs * hs;
    const double a = s / theta, b = omc / t2, c = (theta - s) / (t2 * theta);
    for (int k = 0; k < 9; ++k) {
      R[k] = (I[k] + a * W[k]) + b * W2[k];
      V[k] = (I[k] + b * W[k]) + c * W2[k];
    }
  }
  double t[3];
  mat_vec(V, xi + 3, t);
  set_iso(T, R, t);
  return true;
}

// se3.cpp:109-120 (re-orthonormalises when the Gram drift exceeds 1e-7)
inline void compose(const double* a, const double* b, double* out) {
  double Ra[9], Rb[9], R[9], t[3];
  rot_of(a, Ra);
  rot_of(b, Rb);
  mat_mul(Ra, Rb, R);
  const double tb[3] = {b[3], b[7], b[11]};
  mat_vec(Ra, tb, t);
  t[0] = t[0] + a[3];
  t[1] = t[1] + a[7];
  t[2] = t[2] + a[11];
  double Rt[9], g[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rt[3 * i + j] = R[3 * j + i];
  mat_mul(Rt, R, g);
  double fro = 0.0;
  for (int k = 0; k < 9; ++k) {
    const double d = g[k] - ((k % 4 == 0) ? 1.0 : 0.0);
    fro += d * d;
  }
  if (std::sqrt(fro) > 1e-7) orthonormalize(R, R);
  set_iso(out, R, t);
}

// se3.cpp:122-127
inline void inverse(const double* T, double* out) {
  double R[9], Rt[9], t[3];
  rot_of(T, R);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rt[3 * i + j] = R[3 * j + i];
  const double tt[3] = {T[3], T[7], T[11]};
  mat_vec(Rt, tt, t);
  for (int k = 0; k < 3; ++k) t[k] = -t[k];
  set_iso(out, Rt, t);
}

// se3.cpp:15 Twist::norm
inline double twist_norm6(const double* g) {
  return std::sqrt((g[0] * g[0] + g[1] * g[1] + g[2] * g[2]) + (g[3] * g[3] + g[4] * g[4] + g[5] * g[5]));
}

}  // namespace kreg_se3
