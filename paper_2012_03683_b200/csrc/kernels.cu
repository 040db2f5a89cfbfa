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
constexpr int kUnitSlots = 32 * kUnitSteps;  // slots per sweep work unit

// Candidate stage, grid over X (requests with full == 0 exit at once).
// Cell id + occupancy count.
__global__ void k_cell_assign(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (!R.full || i >= R.n_x) return;
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
}

// Scatter into cell ranges (arbitrary order inside a cell); the count array
// is consumed back to zero so it needs no clearing before the next build.
__global__ void k_scatter(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (!R.full || i >= R.n_x) return;
  const int cell = R.cell_of[i];
  const int slot = atomicSub(&R.cell_count[cell], 1) - 1;
  R.tmp_items[R.cell_start[cell] + slot] = i;
}

// Deterministic order inside a cell: rank = number of smaller indices.
__global__ void k_rank(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (!R.full || s >= R.n_x) return;
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

// ---------------------------------------- exclusive scan of the cell counts
// cell_count (int32, n_cells) -> cell_start (int32, n_cells + 1), three
// launches (tile sums, tile prefix, apply) over 2048-cell tiles.
constexpr int kScanThreads = 256;
constexpr int kScanPerThread = kScanTile / kScanThreads;

__global__ void k_scan_tiles(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const long long base = (long long)blockIdx.x * kScanTile;
  if (!R.full || base >= R.n_cells) return;
  long long s = 0;
  for (int k = 0; k < kScanPerThread; ++k) {
    const long long idx = base + (long long)k * kScanThreads + threadIdx.x;
    if (idx < R.n_cells) s += R.cell_count[idx];
  }
  long long tot;
  block_excl_scan<long long>(s, &tot);
  if (threadIdx.x == 0) R.scan_tiles[blockIdx.x] = tot;
}

__global__ void k_scan_tile_prefix(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.x];
  if (!R.full) return;
  const long long nt = (R.n_cells + kScanTile - 1) / kScanTile;
  long long carry = 0;
  for (long long b = 0; b < nt; b += blockDim.x) {
    const long long t = b + threadIdx.x;
    const long long val = t < nt ? R.scan_tiles[t] : 0;
    long long tot;
    const long long ex = block_excl_scan<long long>(val, &tot);
    if (t < nt) R.scan_tiles[t] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) R.cell_start[R.n_cells] = (int)carry;
}

__global__ void k_scan_apply(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const long long base = (long long)blockIdx.x * kScanTile;
  if (!R.full || base >= R.n_cells) return;
  const long long seg = base + (long long)threadIdx.x * kScanPerThread;
  int vals[kScanPerThread];
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const long long idx = seg + k;
    vals[k] = idx < R.n_cells ? R.cell_count[idx] : 0;
    s += vals[k];
  }
  long long tot;
  long long run = block_excl_scan<long long>(s, &tot) + R.scan_tiles[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const long long idx = seg + k;
    if (idx < R.n_cells) R.cell_start[idx] = (int)run;
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

// Candidate search, one warp per source point j: the 27-cell stencil around
// Ts z_j is 9 contiguous x-rows of the dense grid; lanes stride over the
// candidates (coalesced FP64 loads), FP64 distance test against R_s
// (kernels.hpp:37-42, inner_product.cpp:69), c_ij, c > c_min (:73).
// EMIT=false writes sup_count[j]; EMIT=true writes j's candidates in stencil
// order, contiguously: tile t = j/32 owns 32 rows of H_t entries (H_t = max
// candidates in the tile), entry(j, k) = sup_off[t] + (j%32) H_t + k.
template <bool EMIT>
__global__ void __launch_bounds__(256) k_pair_pass(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (!R.full || j >= R.n_z) return;
  if (EMIT && R.sup_off[R.n_tiles] > R.sup_capacity) return;  // host grows and re-runs
  __shared__ __align__(16) float zf_s[8][kMaxFeat];
  float* zf = zf_s[threadIdx.x >> 5];
  const int fs = R.cp.fstride;
  for (int d = lane; d < fs; d += 32) zf[d] = R.zfeat[(long long)j * fs + d];
  __syncwarp();

  double qx, qy, qz;
  apply_T(R.Ts, R.zx[j], R.zy[j], R.zz[j], qx, qy, qz);
  const long long cxl = (long long)floor((qx - R.origin[0]) * R.inv_h);
  const long long cyl = (long long)floor((qy - R.origin[1]) * R.inv_h);
  const long long czl = (long long)floor((qz - R.origin[2]) * R.inv_h);

  long long out = 0;
  if (EMIT) {
    const long long t0 = R.sup_off[j >> 5], H = (R.sup_off[(j >> 5) + 1] - t0) >> 5;
    out = t0 + (j & 31) * H;
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
            if (dx * dx + dy2 * dy2 + dz2 * dz2 <= R.sup_cutoff_sq) {
              i = R.cell_items[s];
              keep = geo ? true : coefficient(R.cp, R.xfeat + (long long)i * fs, zf, &lc);
            }
          }
          const unsigned m = __ballot_sync(0xffffffffu, keep);
          if (EMIT && keep) {
            const int pos = __popc(m & ((1u << lane) - 1u));
            R.sup[out + cnt + pos] = make_int2(i, __float_as_int(lc));
          }
          cnt += __popc(m);
        }
      }
    }
  }
  if (!EMIT && lane == 0) R.sup_count[j] = cnt;
}

// Tile offsets, one block per request (grid.x = requests):
//  SUP:  candidate list, column height = max candidates in the tile
//        -> sup_off = 32 x prefix; status[3, 4] = {overflow, entries}.
//  !SUP: sweep list, column height = max degree rounded up to whole sweep
//        units of kUnitSteps steps (>= 1 unit so the sweep also visits
//        isolated sources for their displacement) -> unit_off, tile_off =
//        kUnitSlots x unit_off, unit_tile[], status {P, overflow, slots,
//        |T - Ts| displacement, invalid}; resets disp_bits.
template <bool SUP>
__global__ void __launch_bounds__(1024) k_tile_offsets(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.x];
  if (SUP && !R.full) return;
  const int* cnt = SUP ? R.sup_count : R.count;
  const int nt = R.n_tiles;
  long long carry = 0, pairs = 0;
  for (int b = 0; b < nt; b += blockDim.x) {
    const int t = b + threadIdx.x;
    long long v = 0;
    if (t < nt) {
      const int j0 = 32 * t, j1 = min(R.n_z, j0 + 32);
      int d = 0;
      for (int j = j0; j < j1; ++j) {
        const int c = cnt[j];
        d = max(d, c);
        pairs += c;
      }
      v = SUP ? d : (d > 0 ? (d + kUnitSteps - 1) / kUnitSteps : 1);
    }
    long long tot;
    const long long ex = carry + block_excl_scan<long long>(v, &tot);
    if (t < nt) {
      if (SUP) {
        R.sup_off[t] = 32 * ex;
      } else {
        R.unit_off[t] = (int)ex;
        R.tile_off[t] = ex * kUnitSlots;
      }
    }
    carry += tot;
  }
  long long P;
  block_excl_scan<long long>(pairs, &P);
  __shared__ unsigned long long dmax_s;
  if (!SUP) {  // max |T z - Ts z|^2 over the filter blocks (bit patterns of non-negative doubles)
    if (threadIdx.x == 0) dmax_s = 0;
    __syncthreads();
    unsigned long long d = 0;
    for (int b = threadIdx.x; b < (R.n_z + 7) / 8; b += blockDim.x) d = R.disp_blk[b] > d ? R.disp_blk[b] : d;
    atomicMax(&dmax_s, d);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (SUP) {
      R.sup_off[nt] = 32 * carry;
      R.status[3] = 32 * carry > R.sup_capacity ? 1.0 : 0.0;
      R.status[4] = (double)(32 * carry);
    } else {
      R.unit_off[nt] = (int)carry;
      R.tile_off[nt] = carry * kUnitSlots;
      R.status[0] = (double)P;
      R.status[1] = carry * kUnitSlots > R.capacity ? 1.0 : 0.0;
      R.status[2] = (double)(carry * kUnitSlots);
      R.status[5] = sqrt(__longlong_as_double((long long)dmax_s));
      R.status[6] = __longlong_as_double((long long)dmax_s) > R.filter_limit_sq ? 1.0 : 0.0;
    }
  }
  if (!SUP && carry * kUnitSlots <= R.capacity) {
    __syncthreads();
    for (int t = threadIdx.x; t < nt; t += blockDim.x)
      for (int u = R.unit_off[t]; u < R.unit_off[t + 1]; ++u) R.unit_tile[u] = t;
  }
}

// Filter stage, one warp per source j (lanes over its candidate row,
// coalesced 8-B entries + gathers of x_i from the L2-resident cloud). Applies
// the reference predicate |x_i - T z_j|^2 <= cutoff^2 in FP64
// (inner_product.cpp:69) with the same operations as a direct search, so the
// kept set is exactly the direct build's set whenever the candidate radius
// covers cutoff + |T z_j - Ts z_j| (checked: COUNT writes the block's max
// displacement to disp_blk[], k_tile_offsets flags a violation).
// EMIT=false: count[j]. EMIT=true: j's slots {x_i fixed point, log2 c} in
// candidate order into its sliced-ELL column (slot(k) = tile_off[t] + 32 k +
// j%32), padded to the tile's unit-rounded column height.
template <bool EMIT>
__global__ void __launch_bounds__(256) k_filter(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j = blockIdx.x * 8 + wid;
  const bool sup_ok = R.sup_off[R.n_tiles] <= R.sup_capacity;
  if (EMIT && (!sup_ok || R.tile_off[R.n_tiles] > R.capacity)) return;  // host grows and re-runs
  const bool active = j < R.n_z;
  double qx = 0, qy = 0, qz = 0;
  if (active) apply_T(R.T, R.zx[j], R.zy[j], R.zz[j], qx, qy, qz);
  if (!EMIT) {
    __shared__ unsigned long long dblk[8];
    unsigned long long d2 = 0;
    if (active) {
      double sx, sy, sz;
      apply_T(R.Ts, R.zx[j], R.zy[j], R.zz[j], sx, sy, sz);
      const double dx = qx - sx, dy = qy - sy, dz = qz - sz;
      d2 = (unsigned long long)__double_as_longlong(dx * dx + dy * dy + dz * dz);
    }
    if (lane == 0) dblk[wid] = d2;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (int w = 0; w < 8; ++w) m = dblk[w] > m ? dblk[w] : m;
      R.disp_blk[blockIdx.x] = m;
    }
  }
  if (!active) return;
  const int t = j >> 5;
  int ds = 0;
  const int2* row = R.sup;
  if (sup_ok) {
    ds = R.sup_count[j];
    const long long t0 = R.sup_off[t], H = (R.sup_off[t + 1] - t0) >> 5;
    row = R.sup + t0 + (j & 31) * H;
  }
  const long long out = EMIT ? R.tile_off[t] + (j & 31) : 0;
  const double c2 = R.cutoff_sq;
  int cnt = 0;
  for (int sb = 0; sb < ds; sb += 32) {
    const int k = sb + lane;
    bool keep = false;
    int2 e = make_int2(0, 0);
    double x = 0, y = 0, z = 0;
    if (k < ds) {
      e = row[k];
      x = R.xx[e.x];
      y = R.xy[e.x];
      z = R.xz[e.x];
      const double dx = x - qx, dy = y - qy, dz = z - qz;
      keep = dx * dx + dy * dy + dz * dz <= c2;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (EMIT && keep) {
      const long long at = out + 32LL * (cnt + __popc(m & ((1u << lane) - 1u)));
      R.slots[at] = make_int4(__double2int_rn((x - R.anchor[0]) * R.qscale),
                              __double2int_rn((y - R.anchor[1]) * R.qscale),
                              __double2int_rn((z - R.anchor[2]) * R.qscale), e.y);
      R.slot_i[at] = e.x;
    }
    cnt += __popc(m);
  }
  if (!EMIT) {
    if (lane == 0) R.count[j] = cnt;
  } else {
    // pad the column to the tile's unit-rounded height: w = ex2(-inf) = 0
    const int height = (R.unit_off[t + 1] - R.unit_off[t]) * kUnitSteps;
    for (int k = cnt + lane; k < height; k += 32) {
      R.slots[out + 32LL * k] = make_int4(0, 0, 0, __float_as_int(-INFINITY));
      R.slot_i[out + 32LL * k] = -1;
    }
  }
}

// ------------------------------------------------------------------ K3
// Packed FP32 pairs (sm_100 FFMA2/FADD2/FMUL2): candidate transforms are
// processed two at a time, one per half of a 64-bit register pair.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(f2_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Fused F + gradient + displacement sweep over the sliced-ELL pair list.
//  * Work unit = one tile of 32 consecutive sources x kUnitSteps degree steps;
//    lane l owns source j = 32 t + l: per-j moments stay in registers, pair
//    slots (tile_off + 32 k + l) load coalesced, and the x gathers of
//    neighbouring sources (Morton order) hit the same lines.
//  * At every tile change a lane computes q = T_m z_j in FP64 for all M
//    candidates -> fixed point (kept as magic - q), and the displacement
//    |T_m z_j - T_b z_j| (inner_product.cpp:238-246); every tile has >= 1 unit.
//  * Per slot and candidate: d = x - q exactly (IADD + FADD with the 1.5*2^23
//    magic), r^2, w = ex2(r^2 kappa + log2 c) on MUFU, W += w, S += w d;
//    candidates run in pairs on FFMA2/FADD2/FMUL2. Per tile: torque +=
//    q_j x S_j (gw = sum_j q_j x S_j since q x x = q x (x - q)).
//  * Units are cut into nblk = ceil(U / kUnitsPerBlock) work blocks, a function
//    of the pair list only; warp w of a work block takes a contiguous unit
//    range. Work-block totals are reduced in FP64 in a fixed order and the
//    last block of the request reduces the work-block partials in a fixed
//    order: bitwise reproducible, independent of grid and batch composition.
__device__ __forceinline__ long long sweep_work_blocks(long long units) {
  const long long b = (units + kUnitsPerBlock - 1) / kUnitsPerBlock;
  return b < 1 ? 1 : (b > kMaxSweepBlocks ? kMaxSweepBlocks : b);
}

// TMA (bulk async copy) + mbarrier helpers: each warp streams its sweep units
// (32 * kUnitSteps contiguous 8-B slots = 2 KB each) through a private ring of
// kSweepStages shared-memory stages, so DRAM/L2 latency of the pair stream is
// hidden behind the x gathers and math of earlier units.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "KREG_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KREG_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr unsigned kStageBytes = kUnitSlots * sizeof(int4);
constexpr size_t kSweepSmem = (size_t)(kSweepThreads / 32) * kSweepStages * kStageBytes +
                              (size_t)(kSweepThreads / 32) * kSweepStages * sizeof(unsigned long long);

// One unit of one sliced-ELL column (lane = source j) for M candidates. The
// unit's 16-B slots {x fixed point, log2 c} are in shared memory (TMA);
// per candidate pair d = x - q (exact, fixed point), w = ex2(r^2 kappa +
// log2 c), W += w and (GRAD) S += w d on FFMA2/FADD2/FMUL2 + 2 MUFU.EX2.
template <int NP, bool GRAD>
__device__ __forceinline__ void sweep_unit(const int4* __restrict__ stage, int lane, const int (&qx)[2 * NP],
                                           const int (&qy)[2 * NP], const int (&qz)[2 * NP], f2_t kap2,
                                           f2_t (&W)[NP], f2_t (&Sx)[NP], f2_t (&Sy)[NP], f2_t (&Sz)[NP]) {
  const f2_t nmag = pk2(-12582912.0f, -12582912.0f);
#pragma unroll
  for (int k = 0; k < kUnitSteps; ++k) {
    const int4 sl = stage[32 * k + lane];  // conflict-free LDS.128
    const float lc = __int_as_float(sl.w);
    const f2_t lc2 = pk2(lc, lc);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int a = 2 * p, b = 2 * p + 1;
      const f2_t dx = add2(pk2(__int_as_float(sl.x + qx[a]), __int_as_float(sl.x + qx[b])), nmag);
      const f2_t dy = add2(pk2(__int_as_float(sl.y + qy[a]), __int_as_float(sl.y + qy[b])), nmag);
      const f2_t dz = add2(pk2(__int_as_float(sl.z + qz[a]), __int_as_float(sl.z + qz[b])), nmag);
      const f2_t r2 = fma2(dz, dz, fma2(dy, dy, mul2(dx, dx)));
      float e0, e1;
      upk2(fma2(r2, kap2, lc2), e0, e1);
      const f2_t w = pk2(ex2_approx(e0), ex2_approx(e1));
      W[p] = add2(W[p], w);
      if (GRAD) {
        Sx[p] = fma2(w, dx, Sx[p]);
        Sy[p] = fma2(w, dy, Sy[p]);
        Sz[p] = fma2(w, dz, Sz[p]);
      }
    }
  }
}

template <int NP, bool GRAD>
__global__ void __launch_bounds__(kSweepThreads, kSweepMinBlocks) k_sweep(const SweepReq* reqs) {
  constexpr int MAXM = 2 * NP;
  constexpr int NV = GRAD ? 7 : 1;  // reduced values per candidate
  constexpr int NW = kSweepThreads / 32;
  // the request descriptor (~1 KB) is staged in shared memory once per block
  __shared__ __align__(16) SweepReq Rs;
  {
    const int4* g = reinterpret_cast<const int4*>(reqs + blockIdx.y);
    int4* s = reinterpret_cast<int4*>(&Rs);
    for (int k = threadIdx.x; k < (int)(sizeof(SweepReq) / 16); k += blockDim.x) s[k] = g[k];
  }
  __syncthreads();
  const SweepReq& R = Rs;
  const int M = R.M;
  // an overflowed build is skipped (its result is discarded by the host);
  // the unit count is passed by the host when the pair list was built earlier
  long long U = R.units;
  if (U < 0) U = R.tile_off[R.n_tiles] <= R.capacity ? (long long)R.unit_off[R.n_tiles] : 0;
  const long long nblk = sweep_work_blocks(U);
  const long long upb = (U + nblk - 1) / nblk;
  const f2_t kap2 = pk2(R.kappa, R.kappa);
  __shared__ double red[NW][MAXM * 7];
  __shared__ unsigned long long dred[NW][MAXM];
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  int4* ring_all = reinterpret_cast<int4*>(dyn_smem);
  unsigned long long* bar_all =
      reinterpret_cast<unsigned long long*>(dyn_smem + (size_t)NW * kSweepStages * kStageBytes);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < NW * kSweepStages) mbar_init(&bar_all[threadIdx.x], 1);
  mbar_fence_init();
  __syncthreads();

  if (blockIdx.x < nblk) {
    f2_t acc[NP][7];
    unsigned long long dmax[MAXM];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int c = 0; c < 7; ++c) acc[p][c] = 0ull;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) dmax[m] = 0ull;

    const long long u0 = blockIdx.x * upb;
    const long long u1 = min(U, u0 + upb);
    const long long upw = (upb + NW - 1) / NW;
    const long long wu0 = min(u1, u0 + wid * upw);
    const int nunits = (int)(min(u1, wu0 + upw) - wu0);
    int4* ring = ring_all + (size_t)wid * kSweepStages * kUnitSlots;
    unsigned long long* bars = bar_all + wid * kSweepStages;
    const int4* src = R.slots + wu0 * kUnitSlots;
    if (lane == 0) {
      for (int s = 0; s < kSweepStages && s < nunits; ++s) {
        mbar_expect_tx(&bars[s], kStageBytes);
        tma_load_1d(ring + s * kUnitSlots, src + (long long)s * kUnitSlots, kStageBytes, &bars[s]);
      }
    }

    int t = -1;
    bool active = false;
    int qx[MAXM], qy[MAXM], qz[MAXM];
    f2_t W[NP], Sx[NP], Sy[NP], Sz[NP];
#pragma unroll
    for (int m = 0; m < MAXM; ++m) qx[m] = qy[m] = qz[m] = (int)kMagic;
#pragma unroll
    for (int p = 0; p < NP; ++p) W[p] = Sx[p] = Sy[p] = Sz[p] = 0ull;

    auto flush_tile = [&]() {
      if (active) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const f2_t fqx = pk2((float)(int)(kMagic - (unsigned)qx[2 * p]), (float)(int)(kMagic - (unsigned)qx[2 * p + 1]));
          const f2_t fqy = pk2((float)(int)(kMagic - (unsigned)qy[2 * p]), (float)(int)(kMagic - (unsigned)qy[2 * p + 1]));
          const f2_t fqz = pk2((float)(int)(kMagic - (unsigned)qz[2 * p]), (float)(int)(kMagic - (unsigned)qz[2 * p + 1]));
          const f2_t neg = pk2(-1.0f, -1.0f);
          acc[p][0] = add2(acc[p][0], W[p]);
          if (GRAD) {
            acc[p][1] = add2(acc[p][1], Sx[p]);
            acc[p][2] = add2(acc[p][2], Sy[p]);
            acc[p][3] = add2(acc[p][3], Sz[p]);
            acc[p][4] = add2(acc[p][4], fma2(mul2(neg, fqz), Sy[p], mul2(fqy, Sz[p])));
            acc[p][5] = add2(acc[p][5], fma2(mul2(neg, fqx), Sz[p], mul2(fqz, Sx[p])));
            acc[p][6] = add2(acc[p][6], fma2(mul2(neg, fqy), Sx[p], mul2(fqx, Sy[p])));
          }
        }
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) W[p] = Sx[p] = Sy[p] = Sz[p] = 0ull;
    };

    int tiles32 = 0;  // unit -> tile for 32 units at a time, one load per lane
    for (int i = 0; i < nunits; ++i) {
      if ((i & 31) == 0) tiles32 = (i + lane < nunits) ? R.unit_tile[wu0 + i + lane] : 0;
      const int tu = __shfl_sync(0xffffffffu, tiles32, i & 31);
      if (tu != t) {
        flush_tile();
        t = tu;
        const int j = t * 32 + lane;
        active = j < R.n_z;
        if (active) {
          const double zx = R.zx[j], zy = R.zy[j], zz = R.zz[j];
          double bx, by, bz;
          apply_T(R.Tb, zx, zy, zz, bx, by, bz);
          const double lim = 536870912.0;  // 2^29 units; X lies within 2^28 of the anchor
#pragma unroll
          for (int m = 0; m < MAXM; ++m) {
            const int mm = m < M ? m : 0;  // padding candidates repeat candidate 0
            double x, y, z;
            apply_T(R.T[mm], zx, zy, zz, x, y, z);
            const double dx = x - bx, dy = y - by, dz = z - bz;
            const unsigned long long d2 = (unsigned long long)__double_as_longlong(dx * dx + dy * dy + dz * dz);
            dmax[m] = d2 > dmax[m] ? d2 : dmax[m];
            qx[m] = (int)(kMagic - (unsigned)__double2int_rn(fmin(fmax((x - R.anchor[0]) * R.qscale, -lim), lim)));
            qy[m] = (int)(kMagic - (unsigned)__double2int_rn(fmin(fmax((y - R.anchor[1]) * R.qscale, -lim), lim)));
            qz[m] = (int)(kMagic - (unsigned)__double2int_rn(fmin(fmax((z - R.anchor[2]) * R.qscale, -lim), lim)));
          }
        }
      }
      const int s = i % kSweepStages;
      mbar_wait(&bars[s], (unsigned)((i / kSweepStages) & 1));
      if (active) sweep_unit<NP, GRAD>(ring + s * kUnitSlots, lane, qx, qy, qz, kap2, W, Sx, Sy, Sz);
      __syncwarp();
      if (lane == 0 && i + kSweepStages < nunits) {  // refill this stage with unit i + stages
        fence_proxy_async();
        mbar_expect_tx(&bars[s], kStageBytes);
        tma_load_1d(ring + s * kUnitSlots, src + (long long)(i + kSweepStages) * kUnitSlots, kStageBytes, &bars[s]);
      }
    }
    flush_tile();

    // deterministic block reduction in FP64; displacement max
#pragma unroll
    for (int p = 0; p < NP; ++p) {
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        float a0 = 0.0f, a1 = 0.0f;
        if (c < NV) upk2(acc[p][c], a0, a1);
        const double s0 = c < NV ? warp_sum_d((double)a0) : 0.0;
        const double s1 = c < NV ? warp_sum_d((double)a1) : 0.0;
        if (lane == 0) {
          red[wid][(2 * p) * 7 + c] = s0;
          red[wid][(2 * p + 1) * 7 + c] = s1;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      unsigned long long d = dmax[m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_down_sync(0xffffffffu, d, o);
        d = other > d ? other : d;
      }
      if (lane == 0) dred[wid][m] = d;
    }
    __syncthreads();
    if (threadIdx.x < M * 7) {
      double s = 0.0;
      for (int w = 0; w < kSweepThreads / 32; ++w) s += red[w][threadIdx.x];
      R.partials[blockIdx.x * (M * 7) + threadIdx.x] = s;
      __threadfence();
    } else if (threadIdx.x >= 64 && threadIdx.x < 64 + M) {
      const int m = threadIdx.x - 64;
      unsigned long long d = 0;
      for (int w = 0; w < kSweepThreads / 32; ++w) d = dred[w][m] > d ? dred[w][m] : d;
      if (d) atomicMax(&R.disp_bits[m], d);
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
  if (n == 0) return;
  int max_nx = 0, max_nz = 0, n_full = 0;
  long long max_cells = 0;
  for (int r = 0; r < n; ++r) {
    max_nz = max(max_nz, h[r].n_z);
    if (!h[r].full) continue;
    ++n_full;
    max_nx = max(max_nx, h[r].n_x);
    max_cells = max(max_cells, h[r].n_cells);
  }
  int launches = 0;
  if (n_full) {  // candidate stage (requests with full == 0 exit at once)
    const int T = 256;
    const dim3 gx(max(1, (max_nx + T - 1) / T), n);
    k_cell_assign<<<gx, T, 0, st>>>(d);
    const unsigned cell_tiles = (unsigned)max(1LL, (max_cells + kScanTile - 1) / kScanTile);
    k_scan_tiles<<<dim3(cell_tiles, n), kScanThreads, 0, st>>>(d);
    k_scan_tile_prefix<<<n, 1024, 0, st>>>(d);
    k_scan_apply<<<dim3(cell_tiles, n), kScanThreads, 0, st>>>(d);
    k_scatter<<<gx, T, 0, st>>>(d);
    k_rank<<<gx, T, 0, st>>>(d);
    const dim3 gz(max(1, (max_nz + 7) / 8), n);
    k_pair_pass<false><<<gz, 256, 0, st>>>(d);
    k_tile_offsets<true><<<n, 1024, 0, st>>>(d);
    k_pair_pass<true><<<gz, 256, 0, st>>>(d);
    launches += 9;
  }
  const dim3 gt(max(1, (max_nz + 7) / 8), n);  // warp per source
  k_filter<false><<<gt, 256, 0, st>>>(d);
  k_tile_offsets<false><<<n, 1024, 0, st>>>(d);
  k_filter<true><<<gt, 256, 0, st>>>(d);
  count_launch(launches + 3);
}

void sweep_batched(const SweepReq* h, const SweepReq* d, int n, int blocks_per_req, cudaStream_t st,
                   cudaEvent_t ev0, cudaEvent_t ev1) {
  if (n == 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_sweep<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    cudaFuncSetAttribute(k_sweep<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    cudaFuncSetAttribute(k_sweep<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    cudaFuncSetAttribute(k_sweep<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    cudaFuncSetAttribute(k_sweep<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    cudaFuncSetAttribute(k_sweep<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    attr_set = true;
  }
  if (ev0) cudaEventRecord(ev0, st);
  // requests arrive grouped: gradient requests first, then F-only ones
  int n_grad = 0;
  while (n_grad < n && h[n_grad].grad) ++n_grad;
  for (int grp = 0; grp < 2; ++grp) {
    const int r0 = grp == 0 ? 0 : n_grad, r1 = grp == 0 ? n_grad : n;
    if (r1 <= r0) continue;
    int max_m = 1;
    for (int r = r0; r < r1; ++r) max_m = max(max_m, h[r].M);
    const dim3 g(blocks_per_req, r1 - r0);
    const SweepReq* dr = d + r0;
    if (grp == 0) {
      if (max_m <= 2) k_sweep<1, true><<<g, kSweepThreads, kSweepSmem, st>>>(dr);
      else if (max_m <= 4) k_sweep<2, true><<<g, kSweepThreads, kSweepSmem, st>>>(dr);
      else k_sweep<4, true><<<g, kSweepThreads, kSweepSmem, st>>>(dr);
    } else {
      if (max_m <= 2) k_sweep<1, false><<<g, kSweepThreads, kSweepSmem, st>>>(dr);
      else if (max_m <= 4) k_sweep<2, false><<<g, kSweepThreads, kSweepSmem, st>>>(dr);
      else k_sweep<4, false><<<g, kSweepThreads, kSweepSmem, st>>>(dr);
    }
    count_launch(1);
  }
  if (ev1) cudaEventRecord(ev1, st);
}

void displacement(const double* zx, const double* zy, const double* zz, int n, const double* d_T2,
                  unsigned long long* d_out, cudaStream_t st) {
  k_displacement<<<(n + 255) / 256, 256, 0, st>>>(zx, zy, zz, n, d_T2, d_out);
  count_launch();
}

long long kernel_launch_count() { return g_launches.load(); }

}  // namespace kreg_dev
