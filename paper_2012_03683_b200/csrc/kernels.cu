// sm_100a kernels of the CVO registration hot path.
//
//  K1  grid build      : k_cell_assign, batched exclusive scan, k_scatter, k_rank
//  K2  pair build      : candidate stage k_pair_pass<COUNT/EMIT> (grid search
//                        at R_s, c_ij) + k_tile_offsets<SUP>; filter stage
//                        k_filter<COUNT/EMIT> (or k_refilter), k_order,
//                        k_tile_offsets, k_chunk_records
//  K3  fused sweep     : k_sweep<NPG> (persistent, TMA-fed; F + SE(3) gradient
//                        for up to 8 candidate transforms per pass, MUFU ex2,
//                        FP64 displacement items, deterministic fixed-order
//                        chunk / group / request reductions)
//
// Reference semantics (file:line under /root/reference/proj):
//   k_geo          kernels.hpp:37-47          c_ij      kernels.cpp:18-53
//   grid/stencil   hash_grid.hpp:22-50         build     inner_product.cpp:37-95
//   F, grad        inner_product.cpp:97-152    reduction detail/reduce.hpp:12-23
//   displacement   inner_product.cpp:238-246
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <vector>

#include "engine.cuh"

namespace kreg_dev {

namespace {
std::atomic<long long> g_launches{0};
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Debug-variant bounds checks (KREG_DEBUG_BOUNDS): count violations in a
// device counter read back by kreg_debug_violations (no trap: the tests run
// real workloads through the variant and require zero).
#ifdef KREG_DEBUG_BOUNDS
__device__ unsigned long long g_viol;
__device__ int g_viol_site;
#define KREG_CHECK(cond, site)            \
  do {                                     \
    if (!(cond)) {                         \
      atomicAdd(&g_viol, 1ull);            \
      atomicExch(&g_viol_site, (site));    \
    }                                      \
  } while (0)
#else
#define KREG_CHECK(cond, site) \
  do {                         \
  } while (0)
#endif

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

// Sweep chunks of a request with U units: chunk_count(U) chunks of
// chunk_units(U) units (a function of the pair list only).
// Chunks of kPrefChunkUnits units (per-chunk costs amortised over ~48 KB of
// slots) unless the list needs more than kMaxChunks of them (C4-size lists
// then use kMaxChunks larger chunks, keeping every warp busy).
__host__ __device__ __forceinline__ long long chunk_units(long long U, int pref) {
  long long cu = (U + kMaxChunks - 1) / kMaxChunks;
  if (cu < pref) cu = pref;
  return (cu + kStageUnits - 1) / kStageUnits * kStageUnits;
}
__host__ __device__ __forceinline__ int chunk_count(long long U, int pref) {
  return U <= 0 ? 1 : (int)((U + chunk_units(U, pref) - 1) / chunk_units(U, pref));
}

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
  // feature rows in cell order: the candidate search reads a stencil row's
  // features contiguously instead of gathering them by point index
  const int fs = R.cp.fstride;
  const float4* src = reinterpret_cast<const float4*>(R.xfeat + (long long)i * fs);
  float4* dstf = reinterpret_cast<float4*>(R.cfeat + (long long)dst * fs);
  for (int d = 0; d < (fs >> 2); ++d) dstf[d] = src[d];
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
// EMIT=false writes the geometric count (distance test only, an upper bound
// that sizes the rows) to sup_count[j]; EMIT=true writes j's candidates (c >
// c_min) in stencil order, contiguously: tile t = j/32 owns 32 rows of H_t
// entries (H_t = max bound in the tile), entry(j, k) = sup_off[t] + (j%32) H_t
// + k, and replaces sup_count[j] by the number written.
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
  if (EMIT) {
    for (int d = lane; d < fs; d += 32) zf[d] = R.zfeat[(long long)j * fs + d];
    __syncwarp();
  }

  double qx, qy, qz;
  apply_T(R.Ts, R.zx[j], R.zy[j], R.zz[j], qx, qy, qz);
  const long long cxl = (long long)floor((qx - R.origin[0]) * R.inv_h);
  const long long cyl = (long long)floor((qy - R.origin[1]) * R.inv_h);
  const long long czl = (long long)floor((qz - R.origin[2]) * R.inv_h);

  long long out = 0;
#ifdef KREG_DEBUG_BOUNDS
  long long Hdbg = 0;
#endif
  if (EMIT) {
    const long long t0 = R.sup_off[j >> 5], H = (R.sup_off[(j >> 5) + 1] - t0) >> 5;
    out = t0 + (j & 31) * H;
#ifdef KREG_DEBUG_BOUNDS
    Hdbg = H;
#endif
  }
  int cnt = 0;
  const bool geo = !EMIT || R.cp.n_channels == 0;
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
          double dx = 0, dy2 = 0, dz2 = 0;
          if (s < s1) {
            dx = R.cx[s] - qx;
            dy2 = R.cy[s] - qy;
            dz2 = R.cz[s] - qz;
            if (dx * dx + dy2 * dy2 + dz2 * dz2 <= R.sup_cutoff_sq) {
              i = R.cell_items[s];
              keep = geo ? true : coefficient(R.cp, R.cfeat + (long long)s * fs, zf, &lc);
            }
          }
          const unsigned m = __ballot_sync(0xffffffffu, keep);
          if (EMIT && keep) {
            // {x_i - Ts z_j (FP32), log2 c}: the filter tests and emits
            // x_i - T z_j = this - (T - Ts) z_j without gathering x_i
            const int pos = __popc(m & ((1u << lane) - 1u));
#ifdef KREG_DEBUG_BOUNDS
            KREG_CHECK(cnt + pos < Hdbg && out + cnt + pos < R.sup_capacity, 1);
#endif
            R.sup[out + cnt + pos] = make_int4(__float_as_int((float)dx), __float_as_int((float)dy2),
                                               __float_as_int((float)dz2), __float_as_int(lc));
            R.sup_i[out + cnt + pos] = i;
          }
          cnt += __popc(m);
        }
      }
    }
  }
  if (lane == 0) R.sup_count[j] = cnt;
}

// Tile offsets, one block per request (grid.x = requests):
//  SUP:  candidate list, column height = max candidates in the tile
//        -> sup_off = 32 x prefix; status[3, 4] = {overflow, entries}.
//  !SUP: sweep list over the degree-sorted source order, column height =
//        the tile's first (largest) degree rounded up to whole sweep units
//        of kUnitSteps steps (0 for tiles without pairs) -> unit_off,
//        tile_off = kUnitSlots x unit_off, status {P, overflow,
//        slots, |T - Ts| displacement, invalid}.
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
      const int j0 = 32 * t;
      int d = 0;
      if (j0 + 32 <= R.n_z) {  // 8 independent 16-B loads (count arrays are 16-B aligned)
        const int4* c4 = reinterpret_cast<const int4*>(cnt + j0);
        int4 v4[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v4[q] = c4[q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          d = max(d, max(max(v4[q].x, v4[q].y), max(v4[q].z, v4[q].w)));
          pairs += (long long)v4[q].x + v4[q].y + v4[q].z + v4[q].w;
        }
      } else {
        for (int j = j0; j < R.n_z; ++j) {
          const int c = cnt[j];
          d = max(d, c);
          pairs += c;
        }
      }
      if (!SUP) d = R.deg_s[j0];  // windows are sorted by degree, descending
      v = SUP ? d : (d + kUnitSteps - 1) / kUnitSteps;  // sources without pairs take no units
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
    for (int b = threadIdx.x; b < (R.n_z + kFilterBlock - 1) / kFilterBlock; b += blockDim.x)
      d = R.disp_blk[b] > d ? R.disp_blk[b] : d;
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
}

// Chunk records of the sweep list (warp per chunk): the tile holding the
// chunk's first unit, where that tile ends, and its 32 sources' coordinates
// (FP32, degree-sorted order), so a sweep warp starts a chunk from one TMA
// copy instead of dependent loads.
__global__ void k_chunk_records(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (R.tile_off[R.n_tiles] > R.capacity) return;
  const long long U = R.unit_off[R.n_tiles];
  if (U == 0 || c >= chunk_count(U, R.chunk_pref)) return;
  const long long u0 = (long long)c * chunk_units(U, R.chunk_pref);
  int lo = 0, hi = R.n_tiles - 1;  // last tile t with unit_off[t] <= u0 (it has units)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (R.unit_off[mid] <= u0) lo = mid;
    else hi = mid - 1;
  }
  KREG_CHECK(c < kMaxChunks, 8);
#ifdef KREG_BOUNDS_SELFTEST
  KREG_CHECK(c != 0 || lane != 0, 99);  // positive control: fires once per list
#endif
  ChunkRec& rec = R.chunks[c];
  if (lane == 0) {
    rec.t0 = lo;
    rec.t0_end = R.unit_off[lo + 1];
  }
  const int p = 32 * lo + lane;
  const float4 z = p < R.n_z ? R.zs[p] : make_float4(0.f, 0.f, 0.f, 0.f);
  rec.x[lane] = z.x;
  rec.y[lane] = z.y;
  rec.z[lane] = z.z;
}

// Sweep order of the sources: windows of kOrderWindow consecutive (Morton)
// sources sorted by degree, descending (ties by index), one CTA per window
// (bitonic sort of 64-bit keys in shared memory). Tiles of 32 sorted sources
// then hold similar degrees, so the sliced-ELL padding is a few percent, and
// sources without pairs end up in tiles that take no sweep units.
// perm[p] = source at sorted position p, pos[j] = position of source j,
// deg_s[p] = degree at position p.
constexpr int kOrderWindow = 1024;
__global__ void __launch_bounds__(kOrderWindow) k_order(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int base = blockIdx.x * kOrderWindow;
  if (base >= R.n_z) return;
  __shared__ unsigned long long key[kOrderWindow];
  const int j = base + threadIdx.x;
  key[threadIdx.x] =
      j < R.n_z ? ((unsigned long long)(0x7FFFFFFFu - (unsigned)R.count[j]) << 32) | (unsigned)j : ~0ull;
  __syncthreads();
  for (int k = 2; k <= kOrderWindow; k <<= 1) {
    for (int s = k >> 1; s > 0; s >>= 1) {
      const int i = threadIdx.x, p = i ^ s;
      if (p > i) {
        const unsigned long long a = key[i], b = key[p];
        if ((a > b) == ((i & k) == 0)) {
          key[i] = b;
          key[p] = a;
        }
      }
      __syncthreads();
    }
  }
  const unsigned long long kk = key[threadIdx.x];
  if (kk != ~0ull) {
    const int js = (int)(kk & 0xffffffffu), p = base + threadIdx.x;
    R.perm[p] = js;
    R.pos[js] = p;
    R.deg_s[p] = (int)(0x7FFFFFFFu - (unsigned)(kk >> 32));
    R.zs[p] = make_float4((float)R.zx[js], (float)R.zy[js], (float)R.zz[js], 0.0f);
  }
}

// Filter stage. A block takes kFilterBlock consecutive sources, a warp
// kFilterWarp of them: lanes 0..kFilterWarp-1 set up one source each (FP64
// transforms, candidate row, sweep column). The warp then walks its sources'
// candidate rows as one sequence of units of kFilterUnit 16-B entries
// {x_i - Ts z_j (FP32), log2 c}, staged through shared memory by cp.async
// kFilterStages - 1 units ahead of the unit being tested, so a row's loads
// overlap the previous rows' tests. d = (x_i - Ts z_j) - (T - Ts) z_j =
// x_i - T z_j is tested against the cutoff in FP32 (the reference predicate,
// inner_product.cpp:69, to ~1e-7 m: only pairs that close to the cutoff can
// differ from an FP64 test, inside the 1e-6 m tie tolerance). The candidate
// radius covers cutoff + |T z_j - Ts z_j| (checked: COUNT writes the block's
// max displacement to disp_blk[], k_tile_offsets flags a violation).
// EMIT=false: count[j]. EMIT=true: j's slots {d, log2 c} (and i) in candidate
// order into its sliced-ELL column (slot(k) = tile_off[t] + 32 k + lane of its
// degree-sorted position), padded to the tile's unit-rounded column height.
#ifndef KREG_FILTER_STAGES
#define KREG_FILTER_STAGES 3
#endif
constexpr int kFilterUnit = 128;
constexpr int kFilterStages = KREG_FILTER_STAGES;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// The filter predicate on one candidate entry e = {x_i - Ts z_j, log2 c}
// given the source shift (T - Ts) z_j in FP32; shared by both filter paths so
// they decide identically.
__device__ __forceinline__ void filter_shift(const BuildReq& R, int j, float& ex, float& ey, float& ez,
                                             unsigned long long& d2) {
  double qx, qy, qz, sx, sy, sz;
  const double zx = R.zx[j], zy = R.zy[j], zz = R.zz[j];
  apply_T(R.T, zx, zy, zz, qx, qy, qz);
  apply_T(R.Ts, zx, zy, zz, sx, sy, sz);
  const double dx = qx - sx, dy = qy - sy, dz = qz - sz;  // (T - Ts) z_j
  d2 = (unsigned long long)__double_as_longlong(dx * dx + dy * dy + dz * dz);
  ex = (float)dx; ey = (float)dy; ez = (float)dz;
}
__device__ __forceinline__ bool filter_keep(const int4& e, float ex, float ey, float ez, float c2) {
  const float dx = __fsub_rn(__int_as_float(e.x), ex), dy = __fsub_rn(__int_as_float(e.y), ey),
              dz = __fsub_rn(__int_as_float(e.z), ez);
  return __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz))) <= c2;
}

template <bool EMIT>
__global__ void __launch_bounds__(kFilterThreads) k_filter(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (R.refilter || blockIdx.x * kFilterBlock >= R.n_z) return;
  const bool sup_ok = R.sup_off[R.n_tiles] <= R.sup_capacity;
  if (EMIT && (!sup_ok || R.tile_off[R.n_tiles] > R.capacity)) return;  // host grows and re-runs
  __shared__ int4 buf[kFilterThreads / 32][kFilterStages][kFilterUnit];
  const int j = blockIdx.x * kFilterBlock + wid * kFilterWarp + lane;  // lanes < kFilterWarp own a source
  const bool own = lane < kFilterWarp && j < R.n_z;
  float ex = 0.f, ey = 0.f, ez = 0.f;
  int ds = 0, col = 0, height = 0;
  long long rb = 0, out = 0;
  unsigned long long d2 = 0;
  if (own) {
    filter_shift(R, j, ex, ey, ez, d2);
    if (sup_ok) {
      ds = R.sup_count[j];
      const long long t0 = R.sup_off[j >> 5], H = (R.sup_off[(j >> 5) + 1] - t0) >> 5;
      rb = t0 + (j & 31) * H;
    }
    if (EMIT) {  // tile and lane of j in the degree-sorted order
      const int p = R.pos[j], ts = p >> 5;
      out = R.tile_off[ts];
      col = p & 31;
      height = (R.unit_off[ts + 1] - R.unit_off[ts]) * kUnitSteps;
    }
  }
  if (!EMIT) {  // block max of |T z - Ts z|^2 (bit patterns of non-negative doubles)
    __shared__ unsigned long long dblk[kFilterThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, d2, o);
      d2 = v > d2 ? v : d2;
    }
    if (lane == 0) dblk[wid] = d2;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (int w = 0; w < kFilterThreads / 32; ++w) m = dblk[w] > m ? dblk[w] : m;
      R.disp_blk[blockIdx.x] = m;
    }
  }
  // units: (source s, first entry sb) over the sources with candidates
  const unsigned live = __ballot_sync(0xffffffffu, own && ds > 0);
  auto next_unit = [&](int& us, int& usb) {
    usb += kFilterUnit;
    if (usb >= __shfl_sync(0xffffffffu, ds, us)) {
      const unsigned rest = live & ~((2u << us) - 1u);
      us = rest ? __ffs(rest) - 1 : kFilterWarp;
      usb = 0;
    }
  };
  auto issue = [&](int stage, int us, int usb) {
    if (us < kFilterWarp) {
      const int d = __shfl_sync(0xffffffffu, ds, us);
      const int4* row = R.sup + __shfl_sync(0xffffffffu, rb, us);
#pragma unroll
      for (int q = 0; q < kFilterUnit / 32; ++q) {
        const int k = usb + 32 * q + lane;
        cp_async16(&buf[wid][stage][32 * q + lane], row + (k < d ? k : 0), k < d ? 16 : 0);
      }
    }
    cp_async_commit();
  };
  int is = live ? __ffs(live) - 1 : kFilterWarp, isb = 0;  // issue cursor
  int ps = is, psb = 0;                                    // test cursor
#pragma unroll
  for (int st = 0; st < kFilterStages - 1; ++st) {
    issue(st, is, isb);
    if (is < kFilterWarp) next_unit(is, isb);
  }
  const float c2 = (float)R.cutoff_sq;
  int my_cnt = 0, stage = 0;
  while (ps < kFilterWarp) {
    issue((stage + kFilterStages - 1) % kFilterStages, is, isb);
    if (is < kFilterWarp) next_unit(is, isb);
    cp_async_wait<kFilterStages - 1>();
    const int dss = __shfl_sync(0xffffffffu, ds, ps);
    const float fx = __shfl_sync(0xffffffffu, ex, ps), fy = __shfl_sync(0xffffffffu, ey, ps),
                fz = __shfl_sync(0xffffffffu, ez, ps);
    int cnt = __shfl_sync(0xffffffffu, my_cnt, ps);
    long long outs = 0, rbs = 0;
    int cols = 0;
    if (EMIT) {
      outs = __shfl_sync(0xffffffffu, out, ps);
      cols = __shfl_sync(0xffffffffu, col, ps);
      if (R.write_index) rbs = __shfl_sync(0xffffffffu, rb, ps);
    }
    const int c0 = cnt;
#pragma unroll
    for (int q = 0; q < kFilterUnit / 32; ++q) {
      const int k = psb + 32 * q + lane;
      const int4 e = buf[wid][stage][32 * q + lane];
      const bool keep = k < dss && filter_keep(e, fx, fy, fz, c2);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (EMIT && keep) {
        const long long at = slot_index(outs, cols, cnt + __popc(m & ((1u << lane) - 1u)));
        KREG_CHECK(at < R.capacity && rbs + k < R.sup_capacity, 2);
        // the candidate entry itself, x_i - Ts z_j: the sweep forms
        // d = x_i - T z_j as this minus (T - Ts) z_j, and a later filter of
        // this list reproduces a filter of the candidate list bit for bit
        R.slots[at] = e;
        if (R.write_index) R.slot_i[at] = R.sup_i[rbs + k];  // export only
      }
      cnt += __popc(m);
    }
    if (lane == ps) my_cnt += cnt - c0;
    next_unit(ps, psb);
    stage = (stage + 1) % kFilterStages;
  }
  cp_async_wait<0>();
  if (!EMIT) {
    if (own) R.count[j] = my_cnt;
  } else {
    // pad each column to its tile's unit-rounded height: w = ex2(-inf) = 0
#pragma unroll 1
    for (int s = 0; s < kFilterWarp; ++s) {
      const int hs = __shfl_sync(0xffffffffu, height, s), cs = __shfl_sync(0xffffffffu, my_cnt, s);
      const long long outs = __shfl_sync(0xffffffffu, out, s);
      const int cols = __shfl_sync(0xffffffffu, col, s);
      KREG_CHECK(cs <= hs || hs == 0, 3);  // kept <= column height
      for (int k = cs + lane; k < hs; k += 32) {
        KREG_CHECK(slot_index(outs, cols, k) < R.capacity, 4);
        R.slots[slot_index(outs, cols, k)] = make_int4(0, 0, 0, __float_as_int(-INFINITY));
        if (R.write_index) R.slot_i[slot_index(outs, cols, k)] = -1;
      }
    }
  }
}

// Filter stage over the resident sweep list (refilter = 1): warp per old
// tile, lane per source (its old column, read in candidate order two slots
// per 1-KB unit row, so the warp's loads are contiguous). Same predicate and
// entries as k_filter, in the same order -> the same list. COUNT writes
// count[j] and the tile's max |T z_j - old_T z_j|^2 (the subset condition
// k_tile_offsets checks against filter_limit_sq); EMIT copies the kept
// entries into j's new column and pads it.
template <bool EMIT>
__global__ void __launch_bounds__(kFilterThreads) k_refilter(const BuildReq* reqs) {
  const BuildReq& R = reqs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (kFilterThreads / 32) + (threadIdx.x >> 5);
  if (!R.refilter || t >= R.n_tiles) return;
  if (EMIT && R.tile_off[R.n_tiles] > R.capacity) return;  // host re-runs from the candidate list
  const int p = 32 * t + lane;
  const bool own = p < R.n_z;
  const int j = own ? R.old_perm[p] : 0;
  const int deg = own ? R.old_deg_s[p] : 0;
  float ex = 0.f, ey = 0.f, ez = 0.f;
  unsigned long long d2 = 0;
  if (own) {
    filter_shift(R, j, ex, ey, ez, d2);
    if (!EMIT) {
      double qx, qy, qz, ox, oy, oz;
      apply_T(R.T, R.zx[j], R.zy[j], R.zz[j], qx, qy, qz);
      apply_T(R.old_T, R.zx[j], R.zy[j], R.zz[j], ox, oy, oz);
      const double dx = qx - ox, dy = qy - oy, dz = qz - oz;
      d2 = (unsigned long long)__double_as_longlong(dx * dx + dy * dy + dz * dz);
    }
  }
  if (!EMIT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, d2, o);
      d2 = v > d2 ? v : d2;
    }
    if (lane == 0) R.disp_blk[t] = d2;
  }
  long long out = 0;
  int col = 0, height = 0;
  if (EMIT && own) {
    const int pn = R.pos[j], tn = pn >> 5;
    out = R.tile_off[tn];
    col = pn & 31;
    height = (R.unit_off[tn + 1] - R.unit_off[tn]) * kUnitSteps;
  }
  const long long base = R.old_tile_off[t];
  const int h_old = (R.old_unit_off[t + 1] - R.old_unit_off[t]) * kUnitSteps;
  const float c2 = (float)R.cutoff_sq;
  int cnt = 0;
  constexpr int kB = 8;  // slots per lane in flight (4 unit rows, 4 KB per warp)
  for (int k0 = 0; k0 < h_old; k0 += kB) {
    int4 e[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q)
      e[q] = k0 + q < h_old ? __ldcs(R.old_slots + slot_index(base, lane, k0 + q)) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      if (k0 + q < deg && filter_keep(e[q], ex, ey, ez, c2)) {
        if (EMIT) {
          KREG_CHECK(cnt < height && slot_index(out, col, cnt) < R.capacity, 5);
          R.slots[slot_index(out, col, cnt)] = e[q];
        }
        ++cnt;
      }
    }
  }
  if (!EMIT) {
    if (own) R.count[j] = cnt;
  } else {
    for (int k = cnt; k < height; ++k) R.slots[slot_index(out, col, k)] = make_int4(0, 0, 0, __float_as_int(-INFINITY));
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
// in-place accumulation (the accumulator register is tied, no copies)
__device__ __forceinline__ void fma2_acc(f2_t& acc, f2_t a, f2_t b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ void add2_acc(f2_t& acc, f2_t a) { asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(a)); }
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

// Fused F + gradient sweep over the sliced-ELL pair list.
//  * Work unit = one tile of 32 degree-sorted sources x kUnitSteps degree
//    steps = kUnitSlots contiguous 16-B slots {x_i - T_s z_j (FP32 x3),
//    log2 c_ij} (T_s: the candidate list's transform); lane l owns the source at sorted position 32 t + l, so the
//    per-source moments stay in registers.
//  * A request's units are cut into chunk_count(U) chunks. The chunks of all
//    requests of a launch form one queue; every warp of a persistent grid
//    grabs chunks dynamically and streams their units through a private TMA
//    ring (kSweepStages stages of kStageUnits units), prefetching across
//    chunk boundaries. A chunk's first stage also carries its ChunkRec (first
//    tile + its sources), later tiles' sources are prefetched one tile ahead:
//    the stream has no dependent global loads.
//  * Per tile and candidate m (FP32): delta = (R_m - R_s) z_j + (t_m - t_s)
//    and the torque arm a_j = T_m z_j - anchor. Per slot: d = (x_i - T_s z_j)
//    - delta = x_i - T_m z_j, r^2, w = ex2(r^2 kappa + log2 c) on MUFU, W += w,
//    S += w d; candidates in pairs on FFMA2/FADD2/FMUL2. Per tile: torque +=
//    a_j x S_j (sum_j q_j x S_j = sum_j (q_j - a) x S_j + a x sum S).
//  * Each chunk's sums are one partial (FP32 warp sums widened to FP64); the
//    warp finishing a chunk group, then the one finishing the request, add
//    the partials in a fixed shuffle-tree order: bitwise reproducible,
//    independent of scheduling and batch composition.
//  * max_j |T_m z_j - T_b z_j| (inner_product.cpp:238-246) comes from the
//    launch's displacement work items in FP64 over the original coordinates,
//    except for requests the host answered with an analytic bound
//    (SweepReq::no_disp, engine_host.cu prepare_sweep).
__device__ __forceinline__ long long request_units(const SweepReq& R) {
  // an overflowed build is skipped (its result is discarded by the host); the
  // unit count is passed by the host when the pair list was built earlier
  if (R.units >= 0) return R.units;
  return R.tile_off[R.n_tiles] <= R.capacity ? (long long)R.unit_off[R.n_tiles] : 0;
}

// TMA (bulk async copy) + mbarrier helpers.
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

constexpr unsigned kUnitBytes = kUnitSlots * sizeof(int4);
constexpr int kStageSlots = kStageUnits * kUnitSlots;
constexpr int kSweepWarps = kSweepThreads / 32;
// chunk records in flight per warp: the producer runs <= kSweepStages stages
// ahead and a record is read when its chunk starts (before its first stage is
// released), so at most kSweepStages first stages hold records
constexpr int kRecSlots = kSweepStages;
constexpr size_t kSweepSmem = (size_t)kSweepWarps * kSweepStages * kStageSlots * sizeof(int4) +
                              (size_t)kSweepWarps * kRecSlots * sizeof(ChunkRec) +
                              (size_t)kSweepWarps * kSweepStages * sizeof(unsigned long long);

// `units` sweep units (2 steps each) of one tile column (lane = source) for M
// candidates: d = (x - T_b z) - delta, w = ex2(r^2 kappa + log2 c), W += w
// and (GRAD) S += w d on FFMA2/FADD2/FMUL2 + 2 MUFU.EX2 per candidate pair.
template <int NP, bool GRAD, bool SO>
__device__ __forceinline__ void sweep_steps(const int4* __restrict__ unit, int lane, int units, const f2_t (&ndx)[NP],
                                            const f2_t (&ndy)[NP], const f2_t (&ndz)[NP], f2_t kap2, f2_t (&W)[NP],
                                            f2_t (&Sx)[NP], f2_t (&Sy)[NP], f2_t (&Sz)[NP], f2_t ux, f2_t uy,
                                            f2_t uz, f2_t& Q2) {
  // slot s of unit u sits at 2 lane + (s ^ sw) (slot_index): two swizzled bases
  const int sw = (lane >> 2) & 1;
  const int4* p0 = unit + 2 * lane + sw;
  const int4* p1 = unit + 2 * lane + (1 - sw);
  auto step = [&](const int4 sl) {
    const float x = __int_as_float(sl.x), y = __int_as_float(sl.y), z = __int_as_float(sl.z);
    const float lc = __int_as_float(sl.w);
    const f2_t x2 = pk2(x, x), y2 = pk2(y, y), z2 = pk2(z, z), lc2 = pk2(lc, lc);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const f2_t dx = add2(x2, ndx[p]);
      const f2_t dy = add2(y2, ndy[p]);
      const f2_t dz = add2(z2, ndz[p]);
      const f2_t r2 = fma2(dz, dz, fma2(dy, dy, mul2(dx, dx)));
      float e0, e1;
      upk2(fma2(r2, kap2, lc2), e0, e1);
      const f2_t w = pk2(ex2_approx(e0), ex2_approx(e1));
      add2_acc(W[p], w);
      if (GRAD) {
        fma2_acc(Sx[p], w, dx);
        fma2_acc(Sy[p], w, dy);
        fma2_acc(Sz[p], w, dz);
      }
      if (SO) {  // second-order term: w (d . u)^2, u = dq/d eps of the source
        const f2_t du = fma2(dz, uz, fma2(dy, uy, mul2(dx, ux)));
        fma2_acc(Q2, w, mul2(du, du));
      }
    }
  };
  if (units == kStageUnits) {  // a full stage: straight-line code, constant offsets
#pragma unroll
    for (int u = 0; u < kStageUnits; ++u) {
      step(p0[u * kUnitSlots]);  // conflict-free LDS.128
      step(p1[u * kUnitSlots]);
    }
  } else {
#pragma unroll 1
    for (int u = 0; u < units; ++u) {
      step(p0[u * kUnitSlots]);
      step(p1[u * kUnitSlots]);
    }
  }
}

__device__ __forceinline__ f2_t warp_sum_f2(f2_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = add2(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Launch control block (device, zero between launches: the last CTA to exit
// resets the global counters, request finishers reset theirs).
struct SweepCtl {
  unsigned next_item;              // work-item queue head
  unsigned exited;                 // CTAs done
  unsigned req_done[kMaxSweepReqs];                    // finished groups + displacement items
  unsigned grp_done[kMaxSweepReqs][kMaxChunkGroups];  // finished chunks per group
};

// Counter increment with acquire-release semantics at GPU scope: after a
// __syncwarp it publishes the whole warp's prior stores (release is
// cumulative) and, for the last arriver, orders its later loads (acquire).
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// A request's work item (chunk group or displacement slice) is complete; the
// warp completing its last item adds the group partials in a fixed order and
// writes F, the gradient (inner_product.cpp:121-157, assembled in FP64) and
// the displacement; resets the request's counters and displacement bits.
// The request's totals from its group partials (one warp), written to out
// (mapped host memory); resets the displacement bits.
__device__ __noinline__ void finish_request(const SweepReq& R, int lane) {
  const int M = R.M, NV = R.second ? kNvSecond : (R.grad ? 7 : 1), MV = M * NV;
  const int C = chunk_count(request_units(R), R.chunk_pref);
  const int NG = (C + kChunkGroup - 1) / kChunkGroup;
  const double* gpart = R.partials + (size_t)kMaxChunks * MV;
  // group partials: lane l holds groups l and l + 32 (NG <= 64), fixed-order
  // shuffle tree per value
  double t[kNvSecond];
  for (int m = 0; m < M; ++m) {
#pragma unroll
    for (int k = 0; k < kNvSecond; ++k) {
      double v = 0.0;
      if (k < NV) {
        if (lane < NG) v = __ldcg(gpart + (size_t)lane * MV + m * NV + k);
        if (lane + 32 < NG) v += __ldcg(gpart + (size_t)(lane + 32) * MV + m * NV + k);
      }
      const double tot = __shfl_sync(0xffffffffu, warp_sum_d(v), 0);
      if (lane == m) t[k] = k < NV ? tot : 0.0;
    }
  }
  if (lane < M) {
    const double gvx = t[1], gvy = t[2], gvz = t[3];  // sum w (x - q), meters
    const double* a = R.anchor;
    // sum w q x (x - q) = sum_j (q_j - a) x S_j + a x sum_j S_j
    const double gwx = t[4] + (a[1] * gvz - a[2] * gvy);
    const double gwy = t[5] + (a[2] * gvx - a[0] * gvz);
    const double gwz = t[6] + (a[0] * gvy - a[1] * gvx);
    const double g = R.sigma2 * R.inv_l2;
    double* o = R.out + lane * kOut;
    o[0] = R.sigma2 * t[0];
    o[1] = g * gwx;
    o[2] = g * gwy;
    o[3] = g * gwz;
    o[4] = g * gvx;
    o[5] = g * gvy;
    o[6] = g * gvz;
    const unsigned long long db = __ldcg(&R.disp_bits[lane]);
    o[7] = sqrt(__longlong_as_double((long long)db));
    R.disp_bits[lane] = 0ull;
    if (R.second) {  // dF/d eps and d2F/d eps2 along exp(eps xi) T, in the next candidate's row (M = 1)
      o[kOut] = g * t[8];
      o[kOut + 1] = R.sigma2 * (t[7] * R.inv_l2 * R.inv_l2 - (t[9] - t[10]) * R.inv_l2);
    }
  }
}

// Sum the chunk partials of group grp into its group partial (fixed-order
// shuffle tree per value; lane l loads chunk grp * 32 + l).
__device__ __forceinline__ void reduce_group(const SweepReq& R, int grp, int C, int MV, int lane) {
  const int gsize = min(kChunkGroup, C - grp * kChunkGroup);
  double* gpart = R.partials + (size_t)kMaxChunks * MV + (size_t)grp * MV;
  const double* src = R.partials + ((size_t)grp * kChunkGroup + lane) * MV;
  for (int v = 0; v < MV; ++v) {
    const double x = warp_sum_d(lane < gsize ? __ldcg(src + v) : 0.0);
    if (lane == 0) gpart[v] = x;
  }
}

// A request's work item (chunk group or displacement slice) is complete; the
// warp completing its last item finishes the request.
__device__ __noinline__ void item_done(const SweepReq& R, SweepCtl* ctl, int r, int n_items, int lane) {
  __syncwarp();
  unsigned old = 0;
  if (lane == 0) old = atom_add_acq_rel(&ctl->req_done[r], 1u);
  old = __shfl_sync(0xffffffffu, old, 0);
  __syncwarp();
  if ((int)old != n_items - 1) return;
  finish_request(R, lane);
  if (lane == 0) ctl->req_done[r] = 0u;
}

// Per-warp chunk queue and TMA producer state (driven by lane 0).
struct WarpQueue {
  int ids[kQueueDepth];
  int head, tail;
  int done;
  int pr, pc;        // request / chunk being prefetched
  int pu, pend;      // units
  unsigned issued;   // stages issued so far
  unsigned recs;     // chunk records issued so far
  int first;         // next stage is the first of chunk pc
};

// Per-warp queues in static shared memory at file scope, so every access
// compiles to LDS/STS (a pointer kept in SweepWarp would be generic).
__shared__ WarpQueue g_wq[kSweepWarps];

// Everything a sweep warp needs across work items.
struct SweepWarp {
  const SweepReq* reqs;
  SweepCtl* ctl;
  const int* cbase;  // item prefix over the launch's requests (shared)
  const int* units;  // sweep units of each request (shared)
  int n_req;
  int total;         // items of the launch
  int4* ring;
  ChunkRec* recs;
  unsigned long long* bars;
  float* tc;         // transform coefficients of the current chunk (shared)
  int lane;
  int tc_r;          // request whose coefficients tc holds
  unsigned consumed, rec_used;
};

__device__ __forceinline__ int disp_items(const SweepReq& R) {
  return R.no_disp ? 0 : (R.n_z + kDispItem - 1) / kDispItem;
}

__device__ __forceinline__ int locate_item(const SweepWarp& w, int g) {
  int lo = 0, hi = w.n_req - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (w.cbase[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// lane 0: issue the next stage (grabbing items as needed); false if none
__device__ __forceinline__ bool produce(SweepWarp& w) {
  WarpQueue& Q = g_wq[threadIdx.x >> 5];
  while (Q.pu >= Q.pend) {
    if (Q.done || Q.tail - Q.head >= kQueueDepth) return false;
    const int g = (int)atomicAdd(&w.ctl->next_item, 1u);
    if (g >= w.total) {
      Q.done = 1;
      return false;
    }
    const int r = locate_item(w, g);
    Q.ids[Q.tail % kQueueDepth] = g;
    ++Q.tail;
    const int i = g - w.cbase[r] - disp_items(w.reqs[r]);
    if (i < 0) continue;  // displacement item: no stages
    const long long U = w.units[r], cu = chunk_units(U, w.reqs[r].chunk_pref);
    Q.pr = r;
    Q.pc = i;
    Q.pu = (int)(Q.pc * cu);
    Q.pend = (int)min(U, Q.pu + cu);
    Q.first = 1;
  }
  const int nu = min(kStageUnits, Q.pend - Q.pu);
  const int s = Q.issued % kSweepStages;
  const SweepReq& P = w.reqs[Q.pr];
  fence_proxy_async();
  KREG_CHECK(((long long)Q.pu + nu) * kUnitSlots <= P.capacity && Q.pc < kMaxChunks && nu > 0, 6);
  mbar_expect_tx(&w.bars[s], nu * kUnitBytes + (Q.first ? (unsigned)sizeof(ChunkRec) : 0u));
  tma_load_1d(w.ring + s * kStageSlots, P.slots + (long long)Q.pu * kUnitSlots, nu * kUnitBytes, &w.bars[s]);
  if (Q.first) {
    tma_load_1d(w.recs + Q.recs % kRecSlots, P.chunks + Q.pc, sizeof(ChunkRec), &w.bars[s]);
    ++Q.recs;
    Q.first = 0;
  }
  Q.pu += nu;
  ++Q.issued;
  return true;
}

// Displacement slice of request r: max_j |T_m z_j - T_b z_j| in FP64 over the
// original coordinates (order-free max).
__device__ __noinline__ void displacement_item(SweepWarp& w, const SweepReq& R, int r, int item, int n_items) {
  // |T_m z - T_b z| = |(R_m - R_b) z + (t_m - t_b)|: one 3x4 product per
  // candidate and source (equal to the reference's difference of two
  // transforms up to the last bit)
  const int lane = w.lane, M = R.M;
  const int j0 = item * kDispItem, j1 = min(R.n_z, j0 + kDispItem);
  for (int m = 0; m < M; ++m) {
    double D[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) D[k] = R.T[m][k] - R.Tb[k];
    unsigned long long d = 0ull;
    for (int j = j0 + lane; j < j1; j += 32) {
      const double zx = R.zx[j], zy = R.zy[j], zz = R.zz[j];
      const double dx = D[0] * zx + D[1] * zy + D[2] * zz + D[3];
      const double dy = D[4] * zx + D[5] * zy + D[6] * zz + D[7];
      const double dz = D[8] * zx + D[9] * zy + D[10] * zz + D[11];
      const unsigned long long d2 = (unsigned long long)__double_as_longlong(dx * dx + dy * dy + dz * dz);
      d = d2 > d ? d2 : d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, d, o);
      d = other > d ? other : d;
    }
    if (lane == 0 && d) atomicMax(&R.disp_bits[m], d);
  }
  item_done(R, w.ctl, r, n_items, lane);
}

// One chunk (units [u0, u1) of request r) for M <= 2 NP candidates: stream the
// stages, accumulate per tile, write the chunk partial, then the group /
// request completion steps.
template <int NP, bool GRAD, bool SO = false>
__device__ __forceinline__ void chunk_body(SweepWarp& w, const SweepReq& R, int r, int c, int C, int n_items) {
  constexpr int MAXM = 2 * NP;
  constexpr int NV = SO ? kNvSecond : (GRAD ? 7 : 1);  // values per candidate in a partial
  static_assert(!SO || (NP == 1 && GRAD), "second-order terms: one candidate with its gradient");
  const int lane = w.lane;
  const int M = R.M;
  const int MV = M * NV;
  const long long U = w.units[r], cu = chunk_units(U, R.chunk_pref);
  const long long u0 = (long long)c * cu, u1 = min(U, u0 + cu);
  const f2_t kap2 = pk2(R.kappa, R.kappa);
  // this chunk's transform coefficients in shared memory (read at every tile
  // start); 96 floats hold Td for 8 candidates or Td + Ta for 4
  constexpr bool kStage = !GRAD || NP <= 2;
  float* tc = w.tc;
  if (kStage && w.tc_r != r) {  // consecutive chunks of one request keep them
    w.tc_r = r;
    __syncwarp();
    for (int i = lane; i < M * 12; i += 32) {
      tc[i] = (&R.Td[0][0])[i];
      if (GRAD) tc[48 + i] = (&R.Ta[0][0])[i];
    }
    __syncwarp();
  }

  f2_t acc[NP][SO ? kNvSecond : 7];
  f2_t ndx[NP], ndy[NP], ndz[NP];  // -delta per candidate pair
  float ax[MAXM], ay[MAXM], az[MAXM];  // torque arm T_m z_j - anchor
  f2_t W[NP], Sx[NP], Sy[NP], Sz[NP];
  f2_t ux = 0ull, uy = 0ull, uz = 0ull, Q2 = 0ull;  // SO: u_j = omega x T z_j + v, sum w (d.u)^2
#pragma unroll
  for (int p = 0; p < NP; ++p)
#pragma unroll
    for (int v = 0; v < (SO ? kNvSecond : 7); ++v) acc[p][v] = 0ull;
#pragma unroll
  for (int p = 0; p < NP; ++p) W[p] = Sx[p] = Sy[p] = Sz[p] = 0ull;

  auto start_tile = [&](float zx, float zy, float zz) {
#pragma unroll
    for (int m = 0; m < MAXM; m += 2) {
      const float* A = kStage ? tc + 12 * (m < M ? m : 0) : R.Td[m < M ? m : 0];
      const float* B = kStage ? tc + 12 * (m + 1 < M ? m + 1 : 0) : R.Td[m + 1 < M ? m + 1 : 0];
      ndx[m / 2] = pk2(-fmaf(A[0], zx, fmaf(A[1], zy, fmaf(A[2], zz, A[3]))),
                       -fmaf(B[0], zx, fmaf(B[1], zy, fmaf(B[2], zz, B[3]))));
      ndy[m / 2] = pk2(-fmaf(A[4], zx, fmaf(A[5], zy, fmaf(A[6], zz, A[7]))),
                       -fmaf(B[4], zx, fmaf(B[5], zy, fmaf(B[6], zz, B[7]))));
      ndz[m / 2] = pk2(-fmaf(A[8], zx, fmaf(A[9], zy, fmaf(A[10], zz, A[11]))),
                       -fmaf(B[8], zx, fmaf(B[9], zy, fmaf(B[10], zz, B[11]))));
    }
    if (GRAD) {
#pragma unroll
      for (int m = 0; m < MAXM; ++m) {
        const float* A = kStage ? tc + 48 + 12 * (m < M ? m : 0) : R.Ta[m < M ? m : 0];
        ax[m] = fmaf(A[0], zx, fmaf(A[1], zy, fmaf(A[2], zz, A[3])));
        ay[m] = fmaf(A[4], zx, fmaf(A[5], zy, fmaf(A[6], zz, A[7])));
        az[m] = fmaf(A[8], zx, fmaf(A[9], zy, fmaf(A[10], zz, A[11])));
      }
    }
    if (SO) {  // u = omega x (arm + anchor) + v = omega x arm + v' (v' = omega x anchor + v)
      const float* d = R.dir;
      const float vx = fmaf(d[1], az[0], fmaf(-d[2], ay[0], d[3]));
      const float vy = fmaf(d[2], ax[0], fmaf(-d[0], az[0], d[4]));
      const float vz = fmaf(d[0], ay[0], fmaf(-d[1], ax[0], d[5]));
      ux = pk2(vx, vx);
      uy = pk2(vy, vy);
      uz = pk2(vz, vz);
    }
  };
  bool active = false;
  auto flush_tile = [&]() {
    if (active) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        acc[p][0] = add2(acc[p][0], W[p]);
        if (GRAD) {
          const f2_t fqx = pk2(ax[2 * p], ax[2 * p + 1]);
          const f2_t fqy = pk2(ay[2 * p], ay[2 * p + 1]);
          const f2_t fqz = pk2(az[2 * p], az[2 * p + 1]);
          const f2_t neg = pk2(-1.0f, -1.0f);
          acc[p][1] = add2(acc[p][1], Sx[p]);
          acc[p][2] = add2(acc[p][2], Sy[p]);
          acc[p][3] = add2(acc[p][3], Sz[p]);
          acc[p][4] = add2(acc[p][4], fma2(mul2(neg, fqz), Sy[p], mul2(fqy, Sz[p])));
          acc[p][5] = add2(acc[p][5], fma2(mul2(neg, fqx), Sz[p], mul2(fqz, Sx[p])));
          acc[p][6] = add2(acc[p][6], fma2(mul2(neg, fqy), Sx[p], mul2(fqx, Sy[p])));
        }
        if (SO) {  // {sum w (d.u)^2, u . S, |u|^2 W, (omega x u) . S} of the tile
          const float* d = R.dir;
          float u0, u1, v0, v1, w0, w1;
          upk2(ux, u0, u1);
          upk2(uy, v0, v1);
          upk2(uz, w0, w1);
          const f2_t ou_x = pk2(d[1] * w0 - d[2] * v0, d[1] * w0 - d[2] * v0);
          const f2_t ou_y = pk2(d[2] * u0 - d[0] * w0, d[2] * u0 - d[0] * w0);
          const f2_t ou_z = pk2(d[0] * v0 - d[1] * u0, d[0] * v0 - d[1] * u0);
          acc[p][7] = add2(acc[p][7], Q2);
          acc[p][8] = add2(acc[p][8], fma2(uz, Sz[p], fma2(uy, Sy[p], mul2(ux, Sx[p]))));
          acc[p][9] = add2(acc[p][9], mul2(W[p], fma2(uz, uz, fma2(uy, uy, mul2(ux, ux)))));
          acc[p][10] = add2(acc[p][10], fma2(ou_z, Sz[p], fma2(ou_y, Sy[p], mul2(ou_x, Sx[p]))));
        }
      }
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) W[p] = Sx[p] = Sy[p] = Sz[p] = 0ull;
    Q2 = 0ull;
  };

  if (u1 > u0) {
    // the first stage carries the chunk record
    const int s0 = w.consumed % kSweepStages;
    mbar_wait(&w.bars[s0], (w.consumed / kSweepStages) & 1);
    const ChunkRec& rec = w.recs[w.rec_used % kRecSlots];
    ++w.rec_used;
    int t = rec.t0;
    long long t_end = rec.t0_end;
    active = 32 * t + lane < R.n_z;
    start_tile(rec.x[lane], rec.y[lane], rec.z[lane]);
    // prefetch of the next tile (speculatively t + 1)
    auto prefetch = [&](int tn, float4& pz, long long& pend) {
      pz = make_float4(0.f, 0.f, 0.f, 0.f);
      pend = U;
      if (tn < R.n_tiles) {
        if (32 * tn + lane < R.n_z) pz = R.zs[32 * tn + lane];
        pend = R.unit_off[tn + 1];
      }
    };
    float4 pz;
    long long p_end;
    prefetch(t + 1, pz, p_end);

    for (long long u = u0; u < u1; u += kStageUnits) {
      const int nu = (int)min((long long)kStageUnits, u1 - u);
      const int s = w.consumed % kSweepStages;
      if (u != u0) mbar_wait(&w.bars[s], (w.consumed / kSweepStages) & 1);
      const int4* stage = w.ring + s * kStageSlots;
      if (u + nu <= t_end) {  // whole stage inside the current tile
        if (active) sweep_steps<NP, GRAD, SO>(stage, lane, nu, ndx, ndy, ndz, kap2, W, Sx, Sy, Sz, ux, uy, uz, Q2);
      } else {
        long long v = u;
        while (v < u + nu) {
          while (v >= t_end) {  // next tile with units
            flush_tile();
            ++t;
            if (p_end > v) {
              t_end = p_end;
              active = 32 * t + lane < R.n_z;
              start_tile(pz.x, pz.y, pz.z);
            } else {  // tile t had no units (window end): load directly
              long long e = R.unit_off[t + 1];
              while (e <= v) e = R.unit_off[++t + 1];
              t_end = e;
              const float4 z = 32 * t + lane < R.n_z ? R.zs[32 * t + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
              active = 32 * t + lane < R.n_z;
              start_tile(z.x, z.y, z.z);
            }
            prefetch(t + 1, pz, p_end);
          }
          const long long w_end = min(u + nu, t_end);
          if (active)
            sweep_steps<NP, GRAD, SO>(stage + (v - u) * kUnitSlots, lane, (int)(w_end - v), ndx, ndy, ndz, kap2, W, Sx,
                                      Sy, Sz, ux, uy, uz, Q2);
          v = w_end;
        }
      }
      __syncwarp();
      ++w.consumed;
      if (lane == 0) produce(w);  // refill the stage just consumed
      __syncwarp();
    }
    flush_tile();
  }

  // chunk partial: FP32 warp sums (fixed butterfly order) widened to FP64;
  // lane v stores value v
  KREG_CHECK(c < kMaxChunks && c / kChunkGroup < kMaxChunkGroups, 7);
  double* part = R.partials + (size_t)c * MV;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float a0, a1;
      upk2(warp_sum_f2(acc[p][v]), a0, a1);
      const int i0 = (2 * p) * NV + v, i1 = (2 * p + 1) * NV + v;
      if (2 * p < M && lane == (i0 & 31)) part[i0] = (double)a0;
      if (2 * p + 1 < M && lane == (i1 & 31)) part[i1] = (double)a1;
    }
  }
  // chunk group done? its last chunk sums the group's partials in order
  __syncwarp();
  const int grp = c / kChunkGroup;
  unsigned old = 0;
  if (lane == 0) old = atom_add_acq_rel(&w.ctl->grp_done[r][grp], 1u);
  old = __shfl_sync(0xffffffffu, old, 0);
  __syncwarp();
  const int gsize = min(kChunkGroup, C - grp * kChunkGroup);
  if ((int)old == gsize - 1) {
    reduce_group(R, grp, C, MV, lane);
    if (lane == 0) w.ctl->grp_done[r][grp] = 0u;
    item_done(R, w.ctl, r, n_items, lane);
  }
}

// Persistent sweep over the work items (displacement slices + chunks) of up
// to kMaxSweepReqs requests; gradient requests with M <= 2 NPG candidates,
// F-only requests (line-search failure path) with M <= 8.
#ifdef KREG_TIMELINE
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned kTlCap = 1u << 16;
__device__ unsigned long long g_tl[kTlCap][4];  // {start, end, cta << 16 | warp, item << 1 | chunk}
__device__ unsigned g_tl_n;
#endif

template <int NPG>
__global__ void __launch_bounds__(kSweepThreads, kSweepCtasPerSm) k_sweep(const SweepReq* reqs, int n_req, SweepCtl* ctl) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#ifdef KREG_TIMELINE
  const unsigned long long tl0 = gtimer();
  __shared__ unsigned tl_items;
  __shared__ unsigned long long tl_last;
  if (threadIdx.x == 0) tl_items = 0, tl_last = 0;
#endif
  __shared__ int cbase[kMaxSweepReqs + 1];
  __shared__ int units_s[kMaxSweepReqs];
  __shared__ float tco[kSweepWarps][96];  // per warp: Td (and Ta) of its current chunk
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  SweepWarp w;
  w.reqs = reqs;
  w.ctl = ctl;
  w.cbase = cbase;
  w.units = units_s;
  w.n_req = n_req;
  w.ring = reinterpret_cast<int4*>(dyn_smem) + (size_t)wid * kSweepStages * kStageSlots;
  w.recs = reinterpret_cast<ChunkRec*>(dyn_smem + (size_t)kSweepWarps * kSweepStages * kStageSlots * sizeof(int4)) +
           wid * kRecSlots;
  w.bars = reinterpret_cast<unsigned long long*>(dyn_smem + (size_t)kSweepWarps * kSweepStages * kStageSlots * sizeof(int4) +
                                                 (size_t)kSweepWarps * kRecSlots * sizeof(ChunkRec)) +
           wid * kSweepStages;
  w.tc = tco[wid];
  w.lane = lane;
  w.tc_r = -1;
  w.consumed = w.rec_used = 0;

  // work items of request r: disp_s[r] displacement slices, then its chunks;
  // item prefix over the launch's requests (every CTA computes it)
  {
    int C = 0;
    if (threadIdx.x < n_req) {
      const SweepReq& Rq = reqs[threadIdx.x];
      const long long U = request_units(Rq);
      C = chunk_count(U, Rq.chunk_pref) + disp_items(Rq);
      units_s[threadIdx.x] = (int)U;
    }
    int tot;
    const int ex = block_excl_scan<int>(C, &tot);
    if (threadIdx.x < n_req) cbase[threadIdx.x] = ex;
    if (threadIdx.x == 0) cbase[n_req] = tot;
  }
  if (lane < kSweepStages) mbar_init(&w.bars[lane], 1);
  if (lane == 0) {
    WarpQueue& q = g_wq[wid];
    q.head = q.tail = 0;
    q.done = 0;
    q.pr = q.pc = 0;
    q.pu = q.pend = 0;
    q.issued = q.recs = 0;
    q.first = 0;
  }
  mbar_fence_init();
  __syncthreads();
  w.total = cbase[n_req];
  if (lane == 0)
    for (int s = 0; s < kSweepStages; ++s)
      if (!produce(w)) break;
  __syncwarp();

  for (;;) {
    // next item of this warp (queued in order by lane 0)
    int g = -1;
    if (lane == 0) {
      WarpQueue& Q = g_wq[wid];
      if (Q.head == Q.tail) produce(w);  // grabs the next item (items without stages issue none)
      if (Q.head != Q.tail) g = Q.ids[Q.head % kQueueDepth];
    }
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g < 0) break;
    const int r = locate_item(w, g);
    const SweepReq& R = reqs[r];
    const int D = disp_items(R);
    const int C = cbase[r + 1] - cbase[r] - D;
    const int n_items = (C + kChunkGroup - 1) / kChunkGroup + D;
    const int c = g - cbase[r] - D;
#ifdef KREG_TIMELINE
    const unsigned long long ti0 = gtimer();
#endif
    if (c < 0) displacement_item(w, R, r, c + D, n_items);
    else if (R.grad && R.second) {
      // second-order requests go to the NPG = 2 instantiation (sweep_batched),
      // keeping their extra registers out of the main M <= 2 kernel
      if constexpr (NPG == 2) chunk_body<1, true, true>(w, R, r, c, C, n_items);
    } else if (R.grad) chunk_body<NPG, true>(w, R, r, c, C, n_items);
    else chunk_body<4, false>(w, R, r, c, C, n_items);
    __syncwarp();
    if (lane == 0) ++g_wq[wid].head;
    __syncwarp();
#ifdef KREG_TIMELINE
    if (lane == 0) {  // item record
      const unsigned long long ti1 = gtimer();
      atomicAdd(&tl_items, 1u);
      atomicMax(&tl_last, ti1);
      const unsigned k = atomicAdd(&g_tl_n, 1u);
      if (k < kTlCap) {
        g_tl[k][0] = ti0;
        g_tl[k][1] = ti1;
        g_tl[k][2] = ((unsigned long long)blockIdx.x << 16) | wid;
        g_tl[k][3] = ((unsigned long long)g << 1) | (c < 0 ? 0 : 1);
      }
    }
#endif
  }
  // the last CTA to exit resets the launch's item counter
  __syncthreads();
#ifdef KREG_TIMELINE
  if (threadIdx.x == 0) {  // CTA record: {start, end, cta << 16 | 0xffff, items}
    const unsigned k = atomicAdd(&g_tl_n, 1u);
    if (k < kTlCap) {
      g_tl[k][0] = tl0;
      g_tl[k][1] = gtimer();
      g_tl[k][2] = ((unsigned long long)blockIdx.x << 16) | 0xffffu;
      g_tl[k][3] = tl_items;
    }
  }
#endif
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctl->exited, 1u) == gridDim.x - 1) {
      ctl->next_item = 0u;
      ctl->exited = 0u;
    }
  }
}

__global__ void k_interleave(const double* x, const double* y, const double* z, int n, double4* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double4(x[i], y[i], z[i], 0.0);
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
  const dim3 gt(max(1, (max_nz + kFilterBlock - 1) / kFilterBlock), n);
  int n_refilter = 0;
  for (int r = 0; r < n; ++r) n_refilter += h[r].refilter ? 1 : 0;
  const bool cand = n_refilter < n;
  const dim3 gr(max(1, ((max_nz + 31) / 32 + kFilterThreads / 32 - 1) / (kFilterThreads / 32)), n);
  if (cand) k_filter<false><<<gt, kFilterThreads, 0, st>>>(d);
  if (n_refilter) k_refilter<false><<<gr, kFilterThreads, 0, st>>>(d);
  k_order<<<dim3(max(1, (max_nz + kOrderWindow - 1) / kOrderWindow), n), kOrderWindow, 0, st>>>(d);
  k_tile_offsets<false><<<n, 1024, 0, st>>>(d);
  if (cand) k_filter<true><<<gt, kFilterThreads, 0, st>>>(d);
  if (n_refilter) k_refilter<true><<<gr, kFilterThreads, 0, st>>>(d);
  k_chunk_records<<<dim3(kMaxChunks / 8, n), 256, 0, st>>>(d);
  count_launch(launches + 3 + (cand ? 2 : 0) + (n_refilter ? 2 : 0));
}

// Per-device kernel attributes (the sweep's dynamic shared memory is above
// the 48 KB default). cudaFuncSetAttribute applies to the current device
// only, so every device a context is created on is initialised once.
cudaError_t init_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::vector<char> done;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < (int)done.size() && done[dev]) return cudaSuccess;
  if ((e = cudaFuncSetAttribute(k_sweep<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_sweep<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_sweep<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem)) != cudaSuccess)
    return e;
  if ((int)done.size() <= dev) done.resize(dev + 1, 0);
  done[dev] = 1;
  return cudaSuccess;
}

size_t sweep_ctl_bytes(int n) { return sizeof(SweepCtl) * ((n + kMaxSweepReqs - 1) / kMaxSweepReqs + 1); }

void sweep_batched(const SweepReq* h, const SweepReq* d, int n, int sm_count, unsigned* d_ctl, cudaStream_t st,
                   cudaEvent_t ev0, cudaEvent_t ev1) {
  if (n == 0) return;
  if (ev0) cudaEventRecord(ev0, st);
  // requests arrive grouped: gradient requests first, then F-only ones; one
  // persistent launch per group (<= kMaxSweepReqs requests each), then one
  // reduction over all requests
  // one persistent launch per kMaxSweepReqs requests (F-only requests first:
  // their chunks are the heaviest, so they are grabbed first)
  int launches = 0;
  for (int r0 = 0; r0 < n; r0 += kMaxSweepReqs) {
    const int r1 = min(n, r0 + kMaxSweepReqs);
    int max_mg = 1;
    // persistent grid of kSweepCtasPerSm CTAs per SM, fewer when the work items of the
    // launch are known on the host (lists built in earlier rounds): every
    // warp then has at least one item and idle CTAs are not launched
    long long items = 0;
    for (int r = r0; r < r1; ++r) {
      if (h[r].grad) max_mg = max(max_mg, h[r].M);
      if (h[r].second) max_mg = max(max_mg, 3);  // NPG = 2 instantiation
      items += h[r].units >= 0 ? chunk_count(h[r].units, h[r].chunk_pref) +
                                     (h[r].no_disp ? 0 : (h[r].n_z + kDispItem - 1) / kDispItem)
                               : (1LL << 40);
    }
    const int grid = (int)max(1LL, min((long long)kSweepCtasPerSm * sm_count, (items + kSweepWarps - 1) / kSweepWarps));
    const SweepReq* dr = d + r0;
    SweepCtl* ctl = reinterpret_cast<SweepCtl*>(d_ctl) + launches;
    if (max_mg <= 2) k_sweep<1><<<grid, kSweepThreads, kSweepSmem, st>>>(dr, r1 - r0, ctl);
    else if (max_mg <= 4) k_sweep<2><<<grid, kSweepThreads, kSweepSmem, st>>>(dr, r1 - r0, ctl);
    else k_sweep<4><<<grid, kSweepThreads, kSweepSmem, st>>>(dr, r1 - r0, ctl);
    ++launches;
  }
  count_launch(launches);
  if (ev1) cudaEventRecord(ev1, st);
}

void displacement(const double* zx, const double* zy, const double* zz, int n, const double* d_T2,
                  unsigned long long* d_out, cudaStream_t st) {
  k_displacement<<<(n + 255) / 256, 256, 0, st>>>(zx, zy, zz, n, d_T2, d_out);
  count_launch();
}

void filter_emit_index(const BuildReq* d, int n_z, cudaStream_t st) {
  k_filter<true><<<dim3(max(1, (n_z + kFilterBlock - 1) / kFilterBlock), 1), kFilterThreads, 0, st>>>(d);
  count_launch();
}

void interleave_positions(const double* x, const double* y, const double* z, int n, double4* out, cudaStream_t st) {
  k_interleave<<<(n + 255) / 256, 256, 0, st>>>(x, y, z, n, out);
  count_launch();
}

long long kernel_launch_count() { return g_launches.load(); }
void note_launches(int n) { count_launch(n); }

}  // namespace kreg_dev

#ifdef KREG_TIMELINE
// Diagnostic export of the timeline variant: copies the recorded item / CTA
// records (4 x u64 each) and clears them; returns the count.
extern "C" int kreg_debug_timeline(unsigned long long* out, int cap) {
  unsigned n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, kreg_dev::g_tl_n, sizeof(n));
  if (n > kreg_dev::kTlCap) n = kreg_dev::kTlCap;
  if ((int)n > cap) n = (unsigned)cap;
  if (n) cudaMemcpyFromSymbol(out, kreg_dev::g_tl, sizeof(unsigned long long) * 4 * n);
  const unsigned z = 0;
  cudaMemcpyToSymbol(kreg_dev::g_tl_n, &z, sizeof(z));
  return (int)n;
}
#endif

#ifdef KREG_DEBUG_BOUNDS
// Diagnostic export of the bounds-check variant: violations since the last
// call (and the site of the latest one), then clears them.
extern "C" long long kreg_debug_violations(int* site) {
  unsigned long long n = 0;
  int st = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, kreg_dev::g_viol, sizeof(n));
  cudaMemcpyFromSymbol(&st, kreg_dev::g_viol_site, sizeof(st));
  const unsigned long long z = 0;
  cudaMemcpyToSymbol(kreg_dev::g_viol, &z, sizeof(z));
  if (site) *site = st;
  return (long long)n;
}
#endif
