// sm_100a kernels of the CVO registration hot path.
//
//  K1  grid build      : k_cell_assign, batched exclusive scan, k_scatter, k_rank
//  K2  pair build      : k_pair_pass<EMIT=false> (count), scan, k_pair_pass<EMIT=true>
//                        (emit (i, log2 c) + chunk table)
//  K3  fused sweep     : k_transform_sources (q = T z in FP64 -> fixed point,
//                        fused max displacement), k_sweep<MAXM> (F + SE(3)
//                        gradient for up to 8 candidate transforms per pass,
//                        MUFU ex2, deterministic FP64 block/grid reduction)
//
// Reference semantics (file:line under /root/reference/proj):
//   k_geo          kernels.hpp:37-47          c_ij      kernels.cpp:18-53
//   grid/stencil   hash_grid.hpp:22-50         build     inner_product.cpp:37-95
//   F, grad        inner_product.cpp:97-152    reduction detail/reduce.hpp:12-23
//   displacement   inner_product.cpp:238-246
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>

#include "engine.cuh"

namespace kreg_dev {

namespace {
std::atomic<long long> g_launches{0};
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void apply_T(const double* T, double x, double y, double z, double& ox,
                                        double& oy, double& oz) {
  // R p + t, row-major 3x4 (se3.cpp:129-131)
  ox = T[0] * x + T[1] * y + T[2] * z + T[3];
  oy = T[4] * x + T[5] * y + T[6] * z + T[7];
  oz = T[8] * x + T[9] * y + T[10] * z + T[11];
}

template <typename V>
__device__ __forceinline__ V warp_incl_scan(V v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread (blockDim multiple of 32,
// <= 1024). Returns the exclusive prefix; *total gets the block total.
template <typename V>
__device__ V block_excl_scan(V v, V* total) {
  __shared__ V warp_tot[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const V inc = warp_incl_scan(v);
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    V t = lane < nw ? warp_tot[lane] : V(0);
    t = warp_incl_scan(t);
    if (lane < nw) warp_tot[lane] = t;
  }
  __syncthreads();
  const V base = wid > 0 ? warp_tot[wid - 1] : V(0);
  *total = warp_tot[nw - 1];
  __syncthreads();
  return base + inc - v;
}

// ------------------------------------------------------------------ K1
// Cell id + occupancy count + fixed-point copy of X for the sweep.
__global__ void k_cell_assign(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R.n_x) return;
  const double x = R.xx[i], y = R.xy[i], z = R.xz[i];
  // hash_grid.hpp:41-43: floor((p - origin) / cell)
  long long cx = (long long)floor((x - R.origin[0]) * R.inv_h);
  long long cy = (long long)floor((y - R.origin[1]) * R.inv_h);
  long long cz = (long long)floor((z - R.origin[2]) * R.inv_h);
  cx = cx < 0 ? 0 : (cx >= R.gx ? R.gx - 1 : cx);
  cy = cy < 0 ? 0 : (cy >= R.gy ? R.gy - 1 : cy);
  cz = cz < 0 ? 0 : (cz >= R.gz ? R.gz - 1 : cz);
  const int cell = (int)((cz * R.gy + cy) * R.gx + cx);
  R.cell_of[i] = cell;
  atomicAdd(&R.cell_count[cell], 1);
  R.xq[i] = make_int4(__double2int_rn((x - R.anchor[0]) * R.qscale),
                      __double2int_rn((y - R.anchor[1]) * R.qscale),
                      __double2int_rn((z - R.anchor[2]) * R.qscale), 0);
}

// Scatter into cell ranges (arbitrary order inside a cell); the count array
// is consumed back to zero so it needs no clearing before the next build.
__global__ void k_scatter(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R.n_x) return;
  const int cell = R.cell_of[i];
  const int slot = atomicSub(&R.cell_count[cell], 1) - 1;
  R.tmp_items[R.cell_start[cell] + slot] = i;
}

// Deterministic order inside a cell: rank = number of smaller indices.
__global__ void k_rank(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= R.n_x) return;
  const int i = R.tmp_items[s];
  const int cell = R.cell_of[i];
  const int b = R.cell_start[cell], e = R.cell_start[cell + 1];
  int rank = 0;
  for (int t = b; t < e; ++t) rank += R.tmp_items[t] < i;
  const int dst = b + rank;
  R.cell_items[dst] = i;
  R.cx[dst] = R.xx[i];
  R.cy[dst] = R.xy[i];
  R.cz[dst] = R.xz[i];
}

// --------------------------------------------------- batched exclusive scan
// mode 0: cell_count (int32, n_cells) -> cell_start (int32, n_cells + 1)
// mode 1: count      (int32, n_z)     -> offsets    (int64, n_z + 1)
// mode 2: tile_slots (int32, n_tiles) -> tile_off   (int64, n_tiles + 1)
// mode 3: tile_units (int32, n_tiles) -> unit_off   (int32, n_tiles + 1)
struct ScanView {
  const int* in;
  long long n;
  int* out32;
  long long* out64;
  long long* tiles;
};

__device__ __forceinline__ ScanView scan_view(const BuildReq& R, int mode) {
  ScanView v;
  v.out32 = nullptr;
  v.out64 = nullptr;
  if (mode == 0) {
    v.in = R.cell_count; v.n = R.n_cells; v.out32 = R.cell_start;
  } else if (mode == 1) {
    v.in = R.count; v.n = R.n_z; v.out64 = R.offsets;
  } else if (mode == 2) {
    v.in = R.tile_slots; v.n = R.n_tiles; v.out64 = R.tile_off;
  } else {
    v.in = R.tile_units; v.n = R.n_tiles; v.out32 = R.unit_off;
  }
  v.tiles = R.scan_tiles + (long long)mode * R.scan_stride;
  return v;
}

constexpr int kScanThreads = 256;
constexpr int kScanPerThread = kScanTile / kScanThreads;

__global__ void k_scan_tiles(const BuildReq* reqs, int mode) {
  const ScanView v = scan_view(reqs[blockIdx.y], mode);
  const long long base = (long long)blockIdx.x * kScanTile;
  if (base >= v.n) return;
  long long s = 0;
  for (int k = 0; k < kScanPerThread; ++k) {
    const long long idx = base + (long long)k * kScanThreads + threadIdx.x;
    if (idx < v.n) s += v.in[idx];
  }
  long long tot;
  block_excl_scan<long long>(s, &tot);
  if (threadIdx.x == 0) v.tiles[blockIdx.x] = tot;
}

__global__ void k_scan_tile_prefix(const BuildReq* reqs, int mode) {
  const ScanView v = scan_view(reqs[blockIdx.x], mode);
  const long long nt = (v.n + kScanTile - 1) / kScanTile;
  long long carry = 0;
  for (long long b = 0; b < nt; b += blockDim.x) {
    const long long t = b + threadIdx.x;
    const long long val = t < nt ? v.tiles[t] : 0;
    long long tot;
    const long long ex = block_excl_scan<long long>(val, &tot);
    if (t < nt) v.tiles[t] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    const BuildReq& R = reqs[blockIdx.x];
    if (v.out32) v.out32[v.n] = (int)carry;
    else v.out64[v.n] = carry;
    if (mode == 1) R.status[0] = (double)carry;  // pairs
    if (mode == 2) {                               // sliced-ELL slots (incl. padding)
      R.status[1] = carry > R.capacity ? 1.0 : 0.0;
      R.status[2] = (double)carry;
    }
  }
}

__global__ void k_scan_apply(const BuildReq* reqs, int mode) {
  const ScanView v = scan_view(reqs[blockIdx.y], mode);
  const long long base = (long long)blockIdx.x * kScanTile;
  if (base >= v.n) return;
  // thread-contiguous segment of kScanPerThread elements
  const long long seg = base + (long long)threadIdx.x * kScanPerThread;
  long long vals[kScanPerThread];
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const long long idx = seg + k;
    vals[k] = idx < v.n ? v.in[idx] : 0;
    s += vals[k];
  }
  long long tot;
  long long run = block_excl_scan<long long>(s, &tot) + v.tiles[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const long long idx = seg + k;
    if (idx < v.n) {
      if (v.out32) v.out32[idx] = (int)run;
      else v.out64[idx] = run;
    }
    run += vals[k];
  }
}

// ------------------------------------------------------------------ K2
// c_ij = prod_k (SE: s^2 exp(-|u-v|^2/(2l^2)) | linear: <u, v>)  (kernels.cpp:18-53),
// FP32, exp on the MUFU pipe; returns log2(c) through *lc (c > 0 on accept).
// Every channel starts on a 16-B boundary and is zero-padded to a multiple of
// 4 floats (cloud upload), so rows stream as float4 and padding adds zero.
__device__ __forceinline__ bool coefficient(const CoeffParams& cp, const float* __restrict__ u,
                                            const float* zf, float* lc) {
  float c = 1.0f;
  for (int k = 0; k < cp.n_channels; ++k) {
    const ChannelDev& ch = cp.ch[k];
    const float4* u4 = reinterpret_cast<const float4*>(u + ch.offset);
    const float4* z4 = reinterpret_cast<const float4*>(zf + ch.offset);
    const int n4 = (ch.dim + 3) >> 2;
    float acc = 0.0f;
    if (ch.linear) {
      for (int d = 0; d < n4; ++d) {
        const float4 a = __ldg(u4 + d), b = z4[d];
        acc = fmaf(a.x, b.x, acc);
        acc = fmaf(a.y, b.y, acc);
        acc = fmaf(a.z, b.z, acc);
        acc = fmaf(a.w, b.w, acc);
      }
      c *= acc;
    } else {
      for (int d = 0; d < n4; ++d) {
        const float4 a = __ldg(u4 + d), b = z4[d];
        const float e0 = a.x - b.x, e1 = a.y - b.y, e2 = a.z - b.z, e3 = a.w - b.w;
        acc = fmaf(e0, e0, acc);
        acc = fmaf(e1, e1, acc);
        acc = fmaf(e2, e2, acc);
        acc = fmaf(e3, e3, acc);
      }
      c *= ch.sigma2 * ex2_approx(acc * ch.kappa);
    }
  }
  *lc = __log2f(c);
  return c > cp.c_min;  // strict; NaN fails (inner_product.cpp:73)
}

constexpr int kMaxFeat = 64;  // max padded feature row handled in registers/smem

// One warp per source point j: 27-cell stencil = 9 contiguous x-rows of the
// dense grid; lanes stride over candidates (coalesced FP64 loads), FP64
// distance test (kernels.hpp:37-42, inner_product.cpp:69), c_ij, c > c_min.
// EMIT=false writes count[j]; EMIT=true writes j's pairs in stencil order
// into its sliced-ELL column: slot(k) = tile_off[j/32] + 32 k + (j%32), and
// pads the column to the tile's max degree with {0, -inf} (w = 0).
template <bool EMIT>
__global__ void __launch_bounds__(256) k_pair_pass(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= R.n_z) return;
  __shared__ __align__(16) float zf_s[8][kMaxFeat];
  float* zf = zf_s[threadIdx.x >> 5];
  const int fs = R.cp.fstride;
  for (int d = lane; d < fs; d += 32) zf[d] = R.zfeat[(long long)j * fs + d];
  __syncwarp();

  double qx, qy, qz;
  apply_T(R.T, R.zx[j], R.zy[j], R.zz[j], qx, qy, qz);
  const long long cxl = (long long)floor((qx - R.origin[0]) * R.inv_h);
  const long long cyl = (long long)floor((qy - R.origin[1]) * R.inv_h);
  const long long czl = (long long)floor((qz - R.origin[2]) * R.inv_h);

  long long out = 0;
  if (EMIT) {
    if (R.tile_off[R.n_tiles] > R.capacity) return;  // host grows and re-runs
    out = R.tile_off[j >> 5] + (j & 31);
  }
  int cnt = 0;
  const bool geo = R.cp.n_channels == 0;
  if (cxl + 1 >= 0 && cxl - 1 < R.gx) {
    const int x_lo = (int)(cxl - 1 < 0 ? 0 : cxl - 1);
    const int x_hi = (int)(cxl + 1 >= R.gx ? R.gx - 1 : cxl + 1);
    for (int dz = -1; dz <= 1; ++dz) {
      const long long cz = czl + dz;
      if (cz < 0 || cz >= R.gz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const long long cy = cyl + dy;
        if (cy < 0 || cy >= R.gy) continue;
        const long long row = (cz * R.gy + cy) * R.gx;
        const int s0 = R.cell_start[row + x_lo];
        const int s1 = R.cell_start[row + x_hi + 1];
        for (int sb = s0; sb < s1; sb += 32) {
          const int s = sb + lane;
          bool keep = false;
          float lc = 0.0f;
          int i = 0;
          if (s < s1) {
            const double dx = R.cx[s] - qx, dy2 = R.cy[s] - qy, dz2 = R.cz[s] - qz;
            if (dx * dx + dy2 * dy2 + dz2 * dz2 <= R.cutoff_sq) {
              i = R.cell_items[s];
              keep = geo ? true : coefficient(R.cp, R.xfeat + (long long)i * fs, zf, &lc);
            }
          }
          const unsigned m = __ballot_sync(0xffffffffu, keep);
          if (EMIT && keep) {
            const int pos = __popc(m & ((1u << lane) - 1u));
            R.pairs[out + 32LL * (cnt + pos)] = make_int2(i, __float_as_int(lc));
          }
          cnt += __popc(m);
        }
      }
    }
  }
  if (!EMIT) {
    if (lane == 0) R.count[j] = cnt;
  } else {
    // pad the column to the tile's max degree: w = ex2(-inf) = 0
    const int dmax = R.tile_deg[j >> 5];
    for (int k = cnt + lane; k < dmax; k += 32) R.pairs[out + 32LL * k] = make_int2(0, __float_as_int(-INFINITY));
  }
}

// Per tile of 32 consecutive sources: max degree, sliced-ELL slot count and
// sweep work units (kUnitSteps degree steps each).
__global__ void k_tile_sizes(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = j >> 5;
  if (t >= R.n_tiles) return;
  int d = j < R.n_z ? R.count[j] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = max(d, __shfl_xor_sync(0xffffffffu, d, o));
  if ((threadIdx.x & 31) == 0) {
    R.tile_deg[t] = d;
    R.tile_slots[t] = 32 * d;
    R.tile_units[t] = (d + kUnitSteps - 1) / kUnitSteps;
  }
}

// unit -> tile table for the sweep
__global__ void k_unit_tiles(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= R.n_tiles || R.tile_off[R.n_tiles] > R.capacity) return;
  for (int u = R.unit_off[t]; u < R.unit_off[t + 1]; ++u) R.unit_tile[u] = t;
}

// ------------------------------------------------------------------ K3
// q = T_m z_j in FP64 -> (magic - fixed point) per candidate; fused max
// displacement |T_m z - T_b z| (inner_product.cpp:238-246).
__global__ void k_transform_sources(const SweepReq* reqs) {
  const SweepReq& R = reqs[blockIdx.y];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = j < R.n_z;
  double zx = 0, zy = 0, zz = 0;
  if (valid) {
    zx = R.zx[j];
    zy = R.zy[j];
    zz = R.zz[j];
  }
  double bx, by, bz;
  apply_T(R.Tb, zx, zy, zz, bx, by, bz);
  const double lim = 536870912.0;  // 2^29 units; X lies within 2^28 of the anchor
  __shared__ unsigned long long warp_max[32];
  for (int m = 0; m < R.M; ++m) {
    double qx, qy, qz;
    apply_T(R.T[m], zx, zy, zz, qx, qy, qz);
    if (valid) {
      const double fx = fmin(fmax((qx - R.anchor[0]) * R.qscale, -lim), lim);
      const double fy = fmin(fmax((qy - R.anchor[1]) * R.qscale, -lim), lim);
      const double fz = fmin(fmax((qz - R.anchor[2]) * R.qscale, -lim), lim);
      R.q[(long long)m * R.n_z + j] =
          make_int4((int)(kMagic - (unsigned)__double2int_rn(fx)), (int)(kMagic - (unsigned)__double2int_rn(fy)),
                    (int)(kMagic - (unsigned)__double2int_rn(fz)), 0);
    }
    const double dx = qx - bx, dy = qy - by, dz = qz - bz;
    unsigned long long d2 = valid ? (unsigned long long)__double_as_longlong(dx * dx + dy * dy + dz * dz) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_down_sync(0xffffffffu, d2, o);
      d2 = other > d2 ? other : d2;
    }
    if ((threadIdx.x & 31) == 0) warp_max[threadIdx.x >> 5] = d2;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long mx = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = warp_max[w] > mx ? warp_max[w] : mx;
      if (mx) atomicMax(&R.disp_bits[m], mx);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Fused F + gradient sweep over the sliced-ELL pair list. Work unit = one tile
// of 32 consecutive sources x kUnitSteps degree steps: lane l owns source
// j = 32 t + l, so per-j moments stay in registers, pair loads are coalesced
// (slot = tile_off + 32 k + l) and the x gathers of neighbouring sources hit
// the same lines. Units are cut into nblk = ceil(U / kUnitsPerBlock) work
// blocks (a function of the pair list only, so results do not depend on the
// physical grid or on batch composition); warp w of a work block takes units
// w, w+8, ... Per pair and candidate: d = x - q exactly in fixed point (IADD +
// FADD via the 1.5*2^23 magic), r^2, w = ex2(r^2 kappa + log2 c) on MUFU,
// W += w, S += w d; per unit: torque += q_j x S_j (gw = sum_j q_j x S_j since
// q x x = q x (x - q)). The 7*M totals of a work block are reduced in FP64 in
// a fixed order; the last block of a request reduces the work-block partials
// in a fixed order.
__device__ __forceinline__ long long sweep_work_blocks(long long units) {
  const long long b = (units + kUnitsPerBlock - 1) / kUnitsPerBlock;
  return b < 1 ? 1 : (b > kMaxSweepBlocks ? kMaxSweepBlocks : b);
}

// kUnitSteps degree steps of one sliced-ELL column (lane = source j) for M
// candidate transforms: loads first (8 coalesced slots, 8 x gathers), then
// per candidate d = x - q (exact, fixed point), w = ex2(r^2 kappa + log2 c).
template <int MAXM, bool FULL>
__device__ __forceinline__ void sweep_steps(const int2* __restrict__ col, int nk, const int4* __restrict__ xq,
                                            const int4 (&qv)[MAXM], int M, float kappa, float (&W)[MAXM],
                                            float (&Sx)[MAXM], float (&Sy)[MAXM], float (&Sz)[MAXM]) {
  int2 pr[kUnitSteps];
#pragma unroll
  for (int k = 0; k < kUnitSteps; ++k) pr[k] = (FULL || k < nk) ? __ldg(col + 32 * k) : make_int2(0, 0);
  int4 xv[kUnitSteps];
#pragma unroll
  for (int k = 0; k < kUnitSteps; ++k) xv[k] = (FULL || k < nk) ? __ldg(xq + pr[k].x) : make_int4(0, 0, 0, 0);
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    if (m < M) {
#pragma unroll
      for (int k = 0; k < kUnitSteps; ++k) {
        if (FULL || k < nk) {
          const float dx = __int_as_float((unsigned)xv[k].x + (unsigned)qv[m].x) - 12582912.0f;
          const float dy = __int_as_float((unsigned)xv[k].y + (unsigned)qv[m].y) - 12582912.0f;
          const float dz = __int_as_float((unsigned)xv[k].z + (unsigned)qv[m].z) - 12582912.0f;
          const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
          const float w = ex2_approx(fmaf(r2, kappa, __int_as_float(pr[k].y)));
          W[m] += w;
          Sx[m] = fmaf(w, dx, Sx[m]);
          Sy[m] = fmaf(w, dy, Sy[m]);
          Sz[m] = fmaf(w, dz, Sz[m]);
        }
      }
    }
  }
}
template <int MAXM>
__global__ void __launch_bounds__(kSweepThreads) k_sweep(const SweepReq* reqs) {
  const SweepReq& R = reqs[blockIdx.y];
  const int M = R.M;
  // an overflowed build is skipped (its result is discarded by the host)
  const long long U = R.tile_off[R.n_tiles] <= R.capacity ? (long long)R.unit_off[R.n_tiles] : 0;
  const long long nblk = sweep_work_blocks(U);
  const long long upb = (U + nblk - 1) / nblk;
  const float kappa = R.kappa;
  __shared__ double red[kSweepThreads / 32][MAXM * 7];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  if (blockIdx.x < nblk) {
    float acc[MAXM][7];
#pragma unroll
    for (int m = 0; m < MAXM; ++m)
#pragma unroll
      for (int c = 0; c < 7; ++c) acc[m][c] = 0.0f;

    const long long u0 = blockIdx.x * upb;
    const long long u1 = min(U, u0 + upb);
    // warp w takes a contiguous unit range, so consecutive units mostly share
    // a tile: per-source moments and q stay in registers across them
    const long long upw = (upb + kSweepThreads / 32 - 1) / (kSweepThreads / 32);
    const long long wu0 = min(u1, u0 + wid * upw);
    const long long wu1 = min(u1, wu0 + upw);
    int t = -1, deg = 0, ubase = 0;
    bool active = false;
    long long col0 = 0;
    int4 qv[MAXM];
    float W[MAXM], Sx[MAXM], Sy[MAXM], Sz[MAXM];
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      qv[m] = make_int4(0, 0, 0, 0);
      W[m] = Sx[m] = Sy[m] = Sz[m] = 0.0f;
    }
    auto flush_tile = [&]() {
      if (active) {
#pragma unroll
        for (int m = 0; m < MAXM; ++m) {
          if (m < M) {
            const float qx = (float)(int)(kMagic - (unsigned)qv[m].x);
            const float qy = (float)(int)(kMagic - (unsigned)qv[m].y);
            const float qz = (float)(int)(kMagic - (unsigned)qv[m].z);
            acc[m][0] += W[m];
            acc[m][1] += Sx[m];
            acc[m][2] += Sy[m];
            acc[m][3] += Sz[m];
            acc[m][4] += qy * Sz[m] - qz * Sy[m];
            acc[m][5] += qz * Sx[m] - qx * Sz[m];
            acc[m][6] += qx * Sy[m] - qy * Sx[m];
          }
        }
      }
#pragma unroll
      for (int m = 0; m < MAXM; ++m) W[m] = Sx[m] = Sy[m] = Sz[m] = 0.0f;
    };
    for (long long u = wu0; u < wu1; ++u) {
      const int tu = R.unit_tile[u];
      if (tu != t) {
        flush_tile();
        t = tu;
        const int j = t * 32 + lane;
        active = j < R.n_z;
        col0 = R.tile_off[t] + lane;
        deg = R.tile_deg[t];
        ubase = R.unit_off[t];
#pragma unroll
        for (int m = 0; m < MAXM; ++m)
          qv[m] = (m < M && active) ? __ldg(R.q + (long long)m * R.n_z + j) : make_int4(0, 0, 0, 0);
      }
      if (!active) continue;  // only lanes past n_z in the last tile
      const int k0 = (int)(u - ubase) * kUnitSteps;
      const int nk = min(kUnitSteps, deg - k0);
      const int2* col = R.pairs + col0 + 32LL * k0;
      if (nk == kUnitSteps) {
        sweep_steps<MAXM, true>(col, kUnitSteps, R.xq, qv, M, kappa, W, Sx, Sy, Sz);
      } else {
        sweep_steps<MAXM, false>(col, nk, R.xq, qv, M, kappa, W, Sx, Sy, Sz);
      }
    }
    flush_tile();
    // deterministic block reduction in FP64
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      if (m < M) {
#pragma unroll
        for (int c = 0; c < 7; ++c) {
          const double s = warp_sum_d((double)acc[m][c]);
          if (lane == 0) red[wid][m * 7 + c] = s;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < M * 7) {
      double s = 0.0;
      for (int w = 0; w < kSweepThreads / 32; ++w) s += red[w][threadIdx.x];
      R.partials[blockIdx.x * (M * 7) + threadIdx.x] = s;
      __threadfence();
    }
  }
  // last physical block of this request reduces the work-block partials
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(R.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  // thread t sums a contiguous range of work blocks, then fixed-order tree
  const long long per = (nblk + kSweepThreads - 1) / kSweepThreads;
  const long long b0 = threadIdx.x * per, b1 = min(nblk, b0 + per);
  for (int m = 0; m < M; ++m) {
    double v[7] = {0, 0, 0, 0, 0, 0, 0};
    for (long long b = b0; b < b1; ++b)
#pragma unroll
      for (int c = 0; c < 7; ++c) v[c] += __ldcg(R.partials + b * (M * 7) + m * 7 + c);
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const double s = warp_sum_d(v[c]);
      if (lane == 0) red[wid][m * 7 + c] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < M) {
    const int m = threadIdx.x;
    double t[7];
    for (int c = 0; c < 7; ++c) {
      double s = 0.0;
      for (int w = 0; w < kSweepThreads / 32; ++w) s += red[w][m * 7 + c];
      t[c] = s;
    }
    const double u = 1.0 / R.qscale;
    const double gvx = t[1] * u, gvy = t[2] * u, gvz = t[3] * u;  // sum w (x - q), meters
    const double* a = R.anchor;
    // sum w q x (x - q) = sum_j (q_j - a) x S_j + a x sum_j S_j
    const double gwx = t[4] * u * u + (a[1] * gvz - a[2] * gvy);
    const double gwy = t[5] * u * u + (a[2] * gvx - a[0] * gvz);
    const double gwz = t[6] * u * u + (a[0] * gvy - a[1] * gvx);
    const double g = R.sigma2 * R.inv_l2;
    double* o = R.out + m * kOut;
    o[0] = R.sigma2 * t[0];
    o[1] = g * gwx;
    o[2] = g * gwy;
    o[3] = g * gwz;
    o[4] = g * gvx;
    o[5] = g * gvy;
    o[6] = g * gvz;
    const unsigned long long db = R.disp_bits[m];
    o[7] = sqrt(__longlong_as_double((long long)db));
    R.disp_bits[m] = 0ull;
  }
  if (threadIdx.x == 0) *R.counter = 0u;
}

__global__ void k_displacement(const double* zx, const double* zy, const double* zz, int n,
                               const double* T2, unsigned long long* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long d2 = 0;
  if (j < n) {
    double ax, ay, az, bx, by, bz;
    apply_T(T2 + 12, zx[j], zy[j], zz[j], ax, ay, az);  // now
    apply_T(T2, zx[j], zy[j], zz[j], bx, by, bz);       // built
    const double dx = ax - bx, dy = ay - by, dz = az - bz;
    d2 = (unsigned long long)__double_as_longlong(dx * dx + dy * dy + dz * dz);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_down_sync(0xffffffffu, d2, o);
    d2 = other > d2 ? other : d2;
  }
  if ((threadIdx.x & 31) == 0 && d2) atomicMax(out, d2);
}

}  // namespace

// -------------------------------------------------------------- launchers
void build_pairs_batched(const BuildReq* h, const BuildReq* d, int n, cudaStream_t st) {
  int max_nx = 0, max_nz = 0;
  long long max_cells = 0;
  for (int r = 0; r < n; ++r) {
    max_nx = max(max_nx, h[r].n_x);
    max_nz = max(max_nz, h[r].n_z);
    max_cells = max(max_cells, h[r].n_cells);
  }
  if (n == 0) return;
  const int T = 256;
  const dim3 gx(max(1, (max_nx + T - 1) / T), n);
  k_cell_assign<<<gx, T, 0, st>>>(d);
  const long long cell_tiles = (max_cells + kScanTile - 1) / kScanTile;
  k_scan_tiles<<<dim3((unsigned)cell_tiles, n), kScanThreads, 0, st>>>(d, 0);
  k_scan_tile_prefix<<<n, 1024, 0, st>>>(d, 0);
  k_scan_apply<<<dim3((unsigned)cell_tiles, n), kScanThreads, 0, st>>>(d, 0);
  k_scatter<<<gx, T, 0, st>>>(d);
  k_rank<<<gx, T, 0, st>>>(d);
  const dim3 gz(max(1, (max_nz + 7) / 8), n);
  k_pair_pass<false><<<gz, 256, 0, st>>>(d);
  const unsigned z_tiles = (unsigned)max(1, (max_nz + kScanTile - 1) / kScanTile);
  k_scan_tiles<<<dim3(z_tiles, n), kScanThreads, 0, st>>>(d, 1);
  k_scan_tile_prefix<<<n, 1024, 0, st>>>(d, 1);
  k_scan_apply<<<dim3(z_tiles, n), kScanThreads, 0, st>>>(d, 1);
  k_tile_sizes<<<dim3(max(1, (max_nz + 255) / 256), n), 256, 0, st>>>(d);
  for (int mode = 2; mode <= 3; ++mode) {
    k_scan_tiles<<<dim3(z_tiles, n), kScanThreads, 0, st>>>(d, mode);
    k_scan_tile_prefix<<<n, 1024, 0, st>>>(d, mode);
    k_scan_apply<<<dim3(z_tiles, n), kScanThreads, 0, st>>>(d, mode);
  }
  k_pair_pass<true><<<gz, 256, 0, st>>>(d);
  k_unit_tiles<<<dim3(max(1, (max_nz / 32 + 256) / 256), n), 256, 0, st>>>(d);
  count_launch(19);
}

void sweep_batched(const SweepReq* h, const SweepReq* d, int n, int blocks_per_req, cudaStream_t st,
                   cudaEvent_t ev0, cudaEvent_t ev1) {
  if (n == 0) return;
  int max_nz = 1, max_m = 1;
  for (int r = 0; r < n; ++r) {
    max_nz = max(max_nz, h[r].n_z);
    max_m = max(max_m, h[r].M);
  }
  k_transform_sources<<<dim3((max_nz + 255) / 256, n), 256, 0, st>>>(d);
  if (ev0) cudaEventRecord(ev0, st);
  const dim3 g(blocks_per_req, n);
  if (max_m <= 1) k_sweep<1><<<g, kSweepThreads, 0, st>>>(d);
  else if (max_m <= 2) k_sweep<2><<<g, kSweepThreads, 0, st>>>(d);
  else if (max_m <= 4) k_sweep<4><<<g, kSweepThreads, 0, st>>>(d);
  else k_sweep<8><<<g, kSweepThreads, 0, st>>>(d);
  if (ev1) cudaEventRecord(ev1, st);
  count_launch(2);
}

void displacement(const double* zx, const double* zy, const double* zz, int n, const double* d_T2,
                  unsigned long long* d_out, cudaStream_t st) {
  k_displacement<<<(n + 255) / 256, 256, 0, st>>>(zx, zy, zz, n, d_T2, d_out);
  count_launch();
}

long long kernel_launch_count() { return g_launches.load(); }

}  // namespace kreg_dev
