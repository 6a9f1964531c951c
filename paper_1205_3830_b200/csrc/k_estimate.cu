// k_estimate.cu — randomised power-iteration estimate of ||A − B P||_2 with B = A[:, J]
// (Table 5 reports ||A − BP||_2; how it was measured is unstated — reading R15:
// fixed-q power iteration on (A − BP)^H (A − BP) from a Philox start vector; reading R16:
// every dot product is compensated (TwoProd via fma + TwoSum, "Dot2"), because the residual is
// 10^-9…10^-16 of ||A|| and plain fp64 would cancel).
//
// Per iteration (HBM-bound: two streaming passes over A_loc):
//   u  = P x          k_px      column-chunk partials, threads over rows t (coalesced down P)
//   w  = A x          k_ax      thread per row i, column splits; A is streamed once
//   y  = w − B u      k_y       merges the partials in fixed order, subtracts B (u_s + u_c), rounds
//   sb = B^H y        k_bhy     one CTA per pivot column, fixed-shape tree merge
//   z  = A^H y − P^H sb  k_z    warp per column j (coalesced down A), rounds; + ||z||^2 partials
// All merges of partial (s, c) accumulators happen in a fixed order, so the estimate is
// deterministic for a given launch shape.
#include <cstdlib>

#include "rid_device.cuh"
#include "rid_internal.h"
#include "rid_tma.cuh"

namespace rid {

// complex Dot2 accumulator: 4 doubles (re.s, re.c, im.s, im.c)
struct cdd {
  dd re, im;
};
__device__ __forceinline__ void cdd_zero(cdd& a) { a.re = {0.0, 0.0}; a.im = {0.0, 0.0}; }
// a += x * y (complex); conj_x: use conj(x)
__device__ __forceinline__ void cdd_mac(cdd& a, double2 x, double2 y, bool conj_x) {
  const double xi = conj_x ? -x.y : x.y;
  dd_add_prod(a.re, x.x, y.x);
  dd_add_prod(a.re, -xi, y.y);
  dd_add_prod(a.im, x.x, y.y);
  dd_add_prod(a.im, xi, y.x);
}
__device__ __forceinline__ void cdd_merge(cdd& a, const cdd& b) {
  dd_merge(a.re, b.re);
  dd_merge(a.im, b.im);
}
__device__ __forceinline__ void cdd_store(double* p, const cdd& a) {
  reinterpret_cast<double4*>(p)[0] = make_double4(a.re.s, a.re.c, a.im.s, a.im.c);
}
__device__ __forceinline__ cdd cdd_load(const double* p) {
  const double4 v = reinterpret_cast<const double4*>(p)[0];
  cdd a;
  a.re = {v.x, v.y};
  a.im = {v.z, v.w};
  return a;
}
__device__ __forceinline__ cdd cdd_shfl_xor(const cdd& a, int m) {
  cdd o;
  o.re.s = __shfl_xor_sync(0xffffffffu, a.re.s, m);
  o.re.c = __shfl_xor_sync(0xffffffffu, a.re.c, m);
  o.im.s = __shfl_xor_sync(0xffffffffu, a.im.s, m);
  o.im.c = __shfl_xor_sync(0xffffffffu, a.im.c, m);
  return o;
}
// tree merge inside a warp; lane 0 holds the fixed-order result
__device__ __forceinline__ void cdd_warp(cdd& a) {
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const cdd o = cdd_shfl_xor(a, m);
    if (((threadIdx.x & 31) & m) == 0) cdd_merge(a, o);
  }
}
__device__ __forceinline__ void dd_warp(dd& a) {
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    dd o;
    o.s = __shfl_xor_sync(0xffffffffu, a.s, m);
    o.c = __shfl_xor_sync(0xffffffffu, a.c, m);
    if (((threadIdx.x & 31) & m) == 0) dd_merge(a, o);
  }
}

// ---- x0 = N(seed, 5, col0 + j, 0) and per-CTA ||x0||^2 partials ------------------------------
__global__ void k_x0(uint64_t seed, int64_t col0, int64_t n_loc, double2* __restrict__ x,
                     double* __restrict__ part) {
  __shared__ dd sred[8];
  dd a = {0.0, 0.0};
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_loc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = rid_normal(seed, 5u, (uint32_t)(col0 + j), 0u);
    x[j] = v;
    dd_add_prod(a, v.x, v.x);
    dd_add_prod(a, v.y, v.y);
  }
  dd_warp(a);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd t = sred[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) dd_merge(t, sred[q]);
    part[2 * blockIdx.x] = t.s;
    part[2 * blockIdx.x + 1] = t.c;
  }
}

// merge nparts dd scalars -> out[0..1]; thread i merges parts i, i+256, ... in order, then a
// fixed-shape tree over the 256 threads (deterministic for a given nparts)
__global__ void __launch_bounds__(256) k_merge_scalar(const double* __restrict__ part, int nparts,
                                                      double* __restrict__ out) {
  __shared__ double ss[256], sc[256];
  dd t = {0.0, 0.0};
  for (int q = threadIdx.x; q < nparts; q += 256) dd_merge(t, dd{part[2 * q], part[2 * q + 1]});
  ss[threadIdx.x] = t.s;
  sc[threadIdx.x] = t.c;
  __syncthreads();
  for (int h = 128; h >= 1; h >>= 1) {
    if (threadIdx.x < h) {
      dd a = {ss[threadIdx.x], sc[threadIdx.x]};
      dd_merge(a, dd{ss[threadIdx.x + h], sc[threadIdx.x + h]});
      ss[threadIdx.x] = a.s;
      sc[threadIdx.x] = a.c;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = ss[0];
    out[1] = sc[0];
  }
}

// x *= 1 / ||v|| where the norm^2 is the dd in nn[0..1] (x = v / ||v||, one division each)
// Also writes est = sqrt(||v||) to est_out (when non-null) — the estimate after this iteration.
// vmax (nullable): atomicMax of max_j |x_j.re| + |x_j.im| (non-negative doubles order like their
// bit patterns), the bound the fixed-offset accumulation of k_ax_tma needs
__device__ __forceinline__ void vmax_update(unsigned long long* vmax, double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0.0) atomicMax(vmax, (unsigned long long)__double_as_longlong(v));
}
__global__ void k_normalise(const double2* __restrict__ v, int64_t n_loc, const double* __restrict__ nn,
                            double2* __restrict__ x, double* __restrict__ est_out,
                            unsigned long long* __restrict__ vmax) {
  const double nv = __dsqrt_rn(__dadd_rn(nn[0], nn[1]));
  if (blockIdx.x == 0 && threadIdx.x == 0 && est_out) est_out[0] = __dsqrt_rn(nv);
  if (!(nv > 0.0)) return;
  double mx = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_loc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = v[j];
    const double2 r = make_double2(__ddiv_rn(a.x, nv), __ddiv_rn(a.y, nv));
    x[j] = r;
    mx = fmax(mx, fabs(r.x) + fabs(r.y));
  }
  if (vmax) vmax_update(vmax, mx);
}


// ---- u partials: part[chunk][t] = sum_{j in chunk} P[t, j] x[j] -------------------------------
__global__ void k_px(const double2* __restrict__ P, int64_t ldp, int64_t k, int64_t n_loc,
                     const double2* __restrict__ x, int64_t chunk, double* __restrict__ part) {
  const int64_t j0 = (int64_t)blockIdx.x * chunk;
  const int64_t j1 = (j0 + chunk < n_loc) ? j0 + chunk : n_loc;
  for (int64_t t = threadIdx.x; t < k; t += blockDim.x) {
    cdd a;
    cdd_zero(a);
    for (int64_t j = j0; j < j1; ++j) cdd_mac(a, P[j * ldp + t], x[j], false);
    cdd_store(part + ((size_t)blockIdx.x * k + t) * 4, a);
  }
}

// merge part[q][i] over q (fixed order) -> out[i] (cdd)
__global__ void k_merge_vec(const double* __restrict__ part, int nparts, int64_t len,
                            double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    cdd a = cdd_load(part + (size_t)i * 4);
    for (int q = 1; q < nparts; ++q) cdd_merge(a, cdd_load(part + ((size_t)q * len + i) * 4));
    cdd_store(out + (size_t)i * 4, a);
  }
}

// the same merge with a warp per output (short vectors, many parts: u = P x's partials): lane l
// merges parts l, l + 32, ... in order, then a fixed-shape butterfly over the lanes
__global__ void k_merge_vec_warp(const double* __restrict__ part, int nparts, int64_t len,
                                 double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= len) return;  // warp-uniform
  cdd a;
  cdd_zero(a);
  for (int q = lane; q < nparts; q += 32) cdd_merge(a, cdd_load(part + ((size_t)q * len + i) * 4));
  cdd_warp(a);
  if (lane == 0) cdd_store(out + (size_t)i * 4, a);
}

// ---- w partials: part[split][i] = sum_{j in split} A[i, j] x[j] -------------------------------
__global__ void __launch_bounds__(256) k_ax(const double2* __restrict__ A, int64_t lda, int64_t m,
                                            int64_t n_loc, const double2* __restrict__ x,
                                            int64_t split_cols, double* __restrict__ part) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * split_cols;
  const int64_t j1 = (j0 + split_cols < n_loc) ? j0 + split_cols : n_loc;
  if (i >= m) return;
  cdd a;
  cdd_zero(a);
  const double2* Ai = A + i;
  int64_t j = j0;
  for (; j + 4 <= j1; j += 4) {
    const double2 a0 = __ldcs(Ai + (j + 0) * lda), a1 = __ldcs(Ai + (j + 1) * lda);
    const double2 a2 = __ldcs(Ai + (j + 2) * lda), a3 = __ldcs(Ai + (j + 3) * lda);
    cdd_mac(a, a0, __ldg(x + j + 0), false);
    cdd_mac(a, a1, __ldg(x + j + 1), false);
    cdd_mac(a, a2, __ldg(x + j + 2), false);
    cdd_mac(a, a3, __ldg(x + j + 3), false);
  }
  for (; j < j1; ++j) cdd_mac(a, __ldcs(Ai + j * lda), __ldg(x + j), false);
  cdd_store(part + ((size_t)blockIdx.y * m + i) * 4, a);
}

// ---- y = round(w - B (u_s + u_c)); w_parts: nparts x m cdd, u: k cdd --------------------------
// CTA = 32 rows (lane = row) x 8 warps; warp w takes t = w, w + 8, ... (coalesced rows of B);
// warp 0 merges the w partials and the eight B u chains in order (fixed shape: deterministic).
__global__ void __launch_bounds__(256) k_y(const double* __restrict__ wpart, int nparts, int64_t m,
                                           const double2* __restrict__ B, int64_t ldb, int64_t k,
                                           const double* __restrict__ u, double2* __restrict__ y,
                                           unsigned long long* __restrict__ vmax) {
  __shared__ double4 sbu[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  cdd bu;
  cdd_zero(bu);
  if (i < m) {
    for (int64_t t = warp; t < k; t += 8) {
      const double2 b = B[t * ldb + i];
      const double4 ut = reinterpret_cast<const double4*>(u)[t];
      const double2 nb = make_double2(-b.x, -b.y);
      cdd_mac(bu, nb, make_double2(ut.x, ut.z), false);  // exact part of B u_s
      cdd_mac(bu, nb, make_double2(ut.y, ut.w), false);  // B u_c
    }
  }
  sbu[warp][lane] = make_double4(bu.re.s, bu.re.c, bu.im.s, bu.im.c);
  __syncthreads();
  double mx = 0.0;
  if (warp == 0 && i < m) {
    cdd a = cdd_load(wpart + (size_t)i * 4);
    for (int q = 1; q < nparts; ++q) cdd_merge(a, cdd_load(wpart + ((size_t)q * m + i) * 4));
#pragma unroll
    for (int w = 0; w < 8; ++w) cdd_merge(a, cdd_load(&sbu[w][lane].x));
    const double2 yi = make_double2(dd_val(a.re), dd_val(a.im));
    y[i] = yi;
    mx = fabs(yi.x) + fabs(yi.y);
  }
  if (vmax && warp == 0) vmax_update(vmax, mx);
}

// ---- sb[t] = sum_i conj(B[i, t]) y[i]; one CTA per t -------------------------------------------
__global__ void __launch_bounds__(256) k_bhy(const double2* __restrict__ B, int64_t ldb, int64_t m,
                                             const double2* __restrict__ y, double* __restrict__ sb) {
  __shared__ double sred[8][4];
  const int64_t t = blockIdx.x;
  cdd a;
  cdd_zero(a);
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) cdd_mac(a, B[t * ldb + i], y[i], true);
  cdd_warp(a);
  if ((threadIdx.x & 31) == 0) cdd_store(&sred[threadIdx.x >> 5][0], a);
  __syncthreads();
  if (threadIdx.x == 0) {
    cdd r = cdd_load(&sred[0][0]);
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) cdd_merge(r, cdd_load(&sred[q][0]));
    cdd_store(sb + (size_t)t * 4, r);
  }
}

// ---- z[j] = round(sum_i conj(A[i,j]) y[i] - sum_t conj(P[t,j]) (sb_s + sb_c)); warp per column;
//      per-CTA ||z||^2 partials ------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_z(const double2* __restrict__ A, int64_t lda, int64_t m,
                                           int64_t n_loc, const double2* __restrict__ y,
                                           const double2* __restrict__ P, int64_t ldp, int64_t k,
                                           const double* __restrict__ sb, double2* __restrict__ z,
                                           double* __restrict__ npart) {
  __shared__ dd sred[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 8 + warp;
  dd nz = {0.0, 0.0};
  if (j < n_loc) {
    cdd a;
    cdd_zero(a);
    const double2* Aj = A + j * lda;
    int64_t i = lane;
    for (; i + 96 < m; i += 128) {
      const double2 a0 = __ldcs(Aj + i), a1 = __ldcs(Aj + i + 32);
      const double2 a2 = __ldcs(Aj + i + 64), a3 = __ldcs(Aj + i + 96);
      cdd_mac(a, a0, __ldg(y + i), true);
      cdd_mac(a, a1, __ldg(y + i + 32), true);
      cdd_mac(a, a2, __ldg(y + i + 64), true);
      cdd_mac(a, a3, __ldg(y + i + 96), true);
    }
    for (; i < m; i += 32) cdd_mac(a, __ldcs(Aj + i), __ldg(y + i), true);
    for (int64_t t = lane; t < k; t += 32) {
      const double2 p = P[j * ldp + t];
      const double4 s = reinterpret_cast<const double4*>(sb)[t];
      const double2 np = make_double2(-p.x, p.y);  // -conj(p)
      cdd_mac(a, np, make_double2(s.x, s.z), false);
      cdd_mac(a, np, make_double2(s.y, s.w), false);
    }
    cdd_warp(a);
    if (lane == 0) {
      const double2 zj = make_double2(dd_val(a.re), dd_val(a.im));
      z[j] = zj;
      dd_add_prod(nz, zj.x, zj.x);
      dd_add_prod(nz, zj.y, zj.y);
    }
  }
  if (lane == 0) sred[warp] = nz;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd t = sred[0];
    for (int q = 1; q < 8; ++q) dd_merge(t, sred[q]);
    npart[2 * blockIdx.x] = t.s;
    npart[2 * blockIdx.x + 1] = t.c;
  }
}

// ---- TMA-fed streaming passes (default; RID_EST_TMA=0 selects k_ax / k_z above) ---------------
// Both passes read A once as boxes of 128 rows x 8 columns (16 KB, cp.async.bulk.tensor, zero-fill
// past m and n_loc) through an NS-stage ring (the x / y values ride along as a one-row box) handed over with mbarriers (one producing thread,
// per-warp release), so the bytes in flight no longer cost registers and the Dot2 arithmetic
// runs from shared memory. Persistent grids: CTA b takes work items b, b + gridDim.x, ... and
// the ring runs on across item boundaries. Same partial layouts and fixed merge orders as above.
// Fixed-offset compensated accumulation (the TMA passes): with B a bound on the sum of |terms|
// an accumulator will ever see and C a power of two >= 4B, the running sum s starts at C and
// stays in [C − B, C + B], so |s| >= 3B >= |p| for every product p and Dekker's Fast2Sum (3 FP64
// operations) is error-free — against TwoSum's 6 in the Dot2 accumulator: 7 instead of 10 FP64
// operations per real product, on the pipe these passes are bound by. The value is (s − C) + c
// with s − C exact (Sterbenz: s ∈ [C/2, 2C]); the error is that of Dot2 scaled by C / Σ|terms|
// (≤ 2^3 · amax·vmax·count / Σ|terms|), i.e. still O(u²)·Σ|terms| — far inside the 1e-10 parity
// bar (reading R16; tested against the Dot2 passes, RID_EST_TMA=0).
struct fdd {
  double s, c;
};
__device__ __forceinline__ void fdd_add_prod(fdd& a, double x, double y) {
  const double p = __dmul_rn(x, y);
  const double pe = __fma_rn(x, y, -p);
  const double t = __dadd_rn(a.s, p);
  const double e = __dsub_rn(p, __dsub_rn(t, a.s));
  a.s = t;
  a.c = __dadd_rn(a.c, __dadd_rn(pe, e));
}
struct cfdd {
  fdd re, im;
};
__device__ __forceinline__ void cfdd_init(cfdd& a, double C) { a.re = {C, 0.0}; a.im = {C, 0.0}; }
__device__ __forceinline__ void cfdd_mac(cfdd& a, double2 x, double2 y, bool conj_x) {
  const double xi = conj_x ? -x.y : x.y;
  fdd_add_prod(a.re, x.x, y.x);
  fdd_add_prod(a.re, -xi, y.y);
  fdd_add_prod(a.im, x.x, y.y);
  fdd_add_prod(a.im, xi, y.x);
}
// back to a Dot2 pair (s − C exact)
__device__ __forceinline__ cdd cfdd_value(const cfdd& a, double C) {
  cdd r;
  r.re = {__dsub_rn(a.re.s, C), a.re.c};
  r.im = {__dsub_rn(a.im.s, C), a.im.c};
  return r;
}
// a power of two >= 4 B, B = 2 · count · amax · vmax (two products per element per accumulator,
// |re·re'| + |im·im'| <= (|re| + |im|)(|re'| + |im'|))
__device__ __forceinline__ double fdd_offset(const unsigned long long* bounds, int64_t count) {
  const double B = 2.0 * (double)count * __longlong_as_double((long long)bounds[0]) *
                   __longlong_as_double((long long)bounds[1]);
  if (!(B > 0.0)) return 1.0;
  return scalbn(1.0, ilogb(B) + 3);  // 2^(ilogb B + 1) > B
}

constexpr int kEstNS = 6;               // ring stages
constexpr int kEstRows = 128;           // complex rows per box
constexpr int kEstBoxA = kEstRows * 8 * 16;  // bytes of one A box (8 columns)


// w partials: item = (row block rb, column split sp); 256 threads: row r = tid & 127, column half
// h = tid >> 7 (columns 4h..4h+3 of every box); the halves merge in order h = 0, 1 at item end.
// Stage = A box + the 8 x values of its columns (128 B, 1D box).
// FIRST (the first iteration): Dot2 accumulators, which need no bound, and the pass records
// amax = max |Re A| + |Im A| into amax_out on the way (no separate pass over A for the bound)
template <bool FIRST>
__global__ void __launch_bounds__(256, 2)
    k_ax_tma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapX,
             int64_t m, int rblocks, int nitems, int64_t split_cols, int64_t n_loc,
             const unsigned long long* __restrict__ bounds, double* __restrict__ part,
             unsigned long long* __restrict__ amax_out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[kEstNS], empty[kEstNS];
  __shared__ double4 shalf[128];  // the h = 1 half's accumulators, merged by h = 0
  constexpr int kStage = kEstBoxA + 128;
  const int tid = threadIdx.x, lane = tid & 31, r = tid & 127, h = tid >> 7;
  if (tid == 0) {
    tma_prefetch_map(&mapA);
    tma_prefetch_map(&mapX);
    for (int s = 0; s < kEstNS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const int my_items = blockIdx.x < nitems ? (nitems - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nb = (int)((split_cols + 7) / 8);  // boxes per item
  const int64_t nq = (int64_t)my_items * nb;
  auto issue = [&](int64_t q) {
    const int it = blockIdx.x + (int)(q / nb) * gridDim.x, b = (int)(q % nb);
    const int rb = it % rblocks, sp = it / rblocks;
    const int s = (int)(q % kEstNS);
    unsigned char* st = smraw + (size_t)s * kStage;
    const int64_t c0 = sp * split_cols + 8 * (int64_t)b;
    mbar_expect_tx(&full[s], kStage);
    tma_box_g2s(st, &mapA, 2 * rb * kEstRows, (int)c0, &full[s]);
    tma_box_g2s(st + kEstBoxA, &mapX, (int)(2 * c0), 0, &full[s]);
  };
  if (tid == 0)
    for (int64_t q = 0; q < kEstNS - 1 && q < nq; ++q) issue(q);
  int64_t q = 0;
  double amx = 0.0;
  for (int ii = 0; ii < my_items; ++ii) {
    const int it = blockIdx.x + ii * gridDim.x;
    const int rb = it % rblocks, sp = it / rblocks;
    const double C = FIRST ? 0.0 : fdd_offset(bounds, split_cols);  // same for every item
    cfdd acc[4];  // one per column slot: four independent dependency chains
    cdd acc1[4];  // FIRST: Dot2
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      cfdd_init(acc[c], C);
      cdd_zero(acc1[c]);
    }
    for (int b = 0; b < nb; ++b, ++q) {
      if (tid == 0 && q + kEstNS - 1 < nq) {
        const int64_t qn = q + kEstNS - 1;
        if (qn >= kEstNS) mbar_wait(&empty[qn % kEstNS], (unsigned)(((qn / kEstNS) - 1) & 1));
        issue(qn);
      }
      const int s = (int)(q % kEstNS);
      mbar_wait(&full[s], (unsigned)((q / kEstNS) & 1));
      const unsigned char* st = smraw + (size_t)s * kStage;
      // columns past the split (only in its last box, past n_loc) were zero-filled by the TMA
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int cc = 4 * h + c;
        const double2 av = *reinterpret_cast<const double2*>(st + (cc * kEstRows + r) * 16);
        const double2 xv = *reinterpret_cast<const double2*>(st + kEstBoxA + cc * 16);
        if (FIRST) {
          cdd_mac(acc1[c], av, xv, false);
          amx = fmax(amx, fabs(av.x) + fabs(av.y));
        } else {
          cfdd_mac(acc[c], av, xv, false);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    cdd a = FIRST ? acc1[0] : cfdd_value(acc[0], C);
#pragma unroll
    for (int c = 1; c < 4; ++c) cdd_merge(a, FIRST ? acc1[c] : cfdd_value(acc[c], C));
    if (h == 1) shalf[r] = make_double4(a.re.s, a.re.c, a.im.s, a.im.c);
    __syncthreads();
    if (h == 0) {
      const double4 o = shalf[r];
      cdd b2;
      b2.re = {o.x, o.y};
      b2.im = {o.z, o.w};
      cdd_merge(a, b2);
      const int64_t i = (int64_t)rb * kEstRows + r;
      if (i < m) cdd_store(part + ((size_t)sp * m + i) * 4, a);
    }
    __syncthreads();
  }
  if (FIRST) vmax_update(amax_out, amx);
}

// z = round(A^H y − P^H sb): item = 8 consecutive columns, warp w owns column 8 item + w; lane
// holds rows lane + 32 u (u < 4) of every box. Stage = A box + the 128 y values of its rows (2 KB,
// 1D box). One dd partial of ||z||^2 per item (npart[item]), as k_z writes per CTA of 8 columns.
__global__ void __launch_bounds__(256, 2)
    k_z_tma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapY,
            int64_t m, int64_t n_loc, int nitems, const double2* __restrict__ P, int64_t ldp,
            int64_t k, const double* __restrict__ sb, double2* __restrict__ z,
            const unsigned long long* __restrict__ bounds, double* __restrict__ npart) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[kEstNS], empty[kEstNS];
  __shared__ dd sred[8];
  constexpr int kStage = kEstBoxA + kEstRows * 16;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    tma_prefetch_map(&mapA);
    tma_prefetch_map(&mapY);
    for (int s = 0; s < kEstNS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const int my_items = blockIdx.x < nitems ? (nitems - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nb = (int)((m + kEstRows - 1) / kEstRows);
  const int64_t nq = (int64_t)my_items * nb;
  auto issue = [&](int64_t q) {
    const int it = blockIdx.x + (int)(q / nb) * gridDim.x, b = (int)(q % nb);
    const int s = (int)(q % kEstNS);
    unsigned char* st = smraw + (size_t)s * kStage;
    mbar_expect_tx(&full[s], kStage);
    tma_box_g2s(st, &mapA, 2 * b * kEstRows, 8 * it, &full[s]);
    tma_box_g2s(st + kEstBoxA, &mapY, 2 * b * kEstRows, 0, &full[s]);
  };
  if (tid == 0)
    for (int64_t q = 0; q < kEstNS - 1 && q < nq; ++q) issue(q);
  int64_t q = 0;
  for (int ii = 0; ii < my_items; ++ii) {
    const int it = blockIdx.x + ii * gridDim.x;
    const int64_t j = 8 * (int64_t)it + warp;
    const double C = fdd_offset(bounds, m);
    cfdd acc[4];  // one per row slot u: four independent dependency chains
#pragma unroll
    for (int u = 0; u < 4; ++u) cfdd_init(acc[u], C);
    for (int b = 0; b < nb; ++b, ++q) {
      if (tid == 0 && q + kEstNS - 1 < nq) {
        const int64_t qn = q + kEstNS - 1;
        if (qn >= kEstNS) mbar_wait(&empty[qn % kEstNS], (unsigned)(((qn / kEstNS) - 1) & 1));
        issue(qn);
      }
      const int s = (int)(q % kEstNS);
      mbar_wait(&full[s], (unsigned)((q / kEstNS) & 1));
      const unsigned char* st = smraw + (size_t)s * kStage;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = lane + 32 * u;
        const double2 av = *reinterpret_cast<const double2*>(st + (warp * kEstRows + rr) * 16);
        const double2 yv = *reinterpret_cast<const double2*>(st + kEstBoxA + rr * 16);
        cfdd_mac(acc[u], av, yv, true);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    cdd a = cfdd_value(acc[0], C);
#pragma unroll
    for (int u = 1; u < 4; ++u) cdd_merge(a, cfdd_value(acc[u], C));
    dd nz = {0.0, 0.0};
    if (j < n_loc) {
      for (int64_t t = lane; t < k; t += 32) {
        const double2 p = P[j * ldp + t];
        const double4 sv = reinterpret_cast<const double4*>(sb)[t];
        const double2 np = make_double2(-p.x, p.y);  // -conj(p)
        cdd_mac(a, np, make_double2(sv.x, sv.z), false);
        cdd_mac(a, np, make_double2(sv.y, sv.w), false);
      }
    }
    cdd_warp(a);
    if (lane == 0 && j < n_loc) {
      const double2 zj = make_double2(dd_val(a.re), dd_val(a.im));
      z[j] = zj;
      dd_add_prod(nz, zj.x, zj.x);
      dd_add_prod(nz, zj.y, zj.y);
    }
    if (lane == 0) sred[warp] = nz;
    __syncthreads();
    if (tid == 0) {
      dd t = sred[0];
      for (int w = 1; w < 8; ++w) dd_merge(t, sred[w]);
      npart[2 * it] = t.s;
      npart[2 * it + 1] = t.c;
    }
    __syncthreads();
  }
}

bool est_tma_enabled() {
  const char* v = select_env("RID_EST_TMA");
  return !(v && atoi(v) == 0);
}

static cudaError_t est_maps(const double2* A, int64_t lda, int64_t m, int64_t n_loc,
                            const double2* v, int64_t vlen, int vbox, CUtensorMap* mapA,
                            CUtensorMap* mapV) {
  PFN_cuTensorMapEncodeTiled encode;
  cudaError_t e = tensor_map_encoder(&encode);
  if (e != cudaSuccess) return e;
  const cuuint32_t estr[2] = {1u, 1u};
  const cuuint64_t gdim[2] = {(cuuint64_t)(2 * m), (cuuint64_t)n_loc};
  const cuuint64_t gstr[1] = {(cuuint64_t)lda * sizeof(double2)};
  const cuuint32_t box[2] = {(cuuint32_t)(2 * kEstRows), 8u};
  if (encode(mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, gdim, gstr, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  // the vector as a one-row 2D tensor (2 vlen doubles x 1)
  const cuuint64_t vdim[2] = {(cuuint64_t)(2 * vlen), 1};
  const cuuint64_t vstr[1] = {(cuuint64_t)((16 * vlen + 15) / 16 * 16)};
  const cuuint32_t vb[2] = {(cuuint32_t)vbox, 1u};
  if (encode(mapV, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)v, vdim, vstr, vb, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

// ------------------------------------------------------------------------------ launchers ------
EstPlan est_plan(int64_t m, int64_t n_loc, int64_t k, int num_sms) {
  EstPlan p;
  p.tma = est_tma_enabled();
  p.px_chunk = 64;
  p.px_parts = (int)((n_loc + p.px_chunk - 1) / p.px_chunk);
  if (p.tma) {
    // work items (row block, column split): >= 12 per CTA slot (2 per SM) for balance
    p.ax_rblocks = (int)((m + kEstRows - 1) / kEstRows);
    int64_t splits = (12 * 2 * (int64_t)num_sms + p.ax_rblocks - 1) / p.ax_rblocks;
    const int64_t cols8 = (n_loc + 7) / 8;
    if (splits > cols8) splits = cols8;
    if (splits > 256) splits = 256;
    if (splits < 1) splits = 1;
    p.ax_split_cols = ((n_loc + splits - 1) / splits + 7) / 8 * 8;
    p.ax_parts = (int)((n_loc + p.ax_split_cols - 1) / p.ax_split_cols);
  } else {
    const int64_t row_blocks = (m + 255) / 256;
    int64_t splits = (8 * num_sms + row_blocks - 1) / row_blocks;
    if (splits < 1) splits = 1;
    if (splits > n_loc) splits = n_loc;
    if (splits > 1024) splits = 1024;
    p.ax_split_cols = (n_loc + splits - 1) / splits;
    p.ax_parts = (int)((n_loc + p.ax_split_cols - 1) / p.ax_split_cols);
    p.ax_rblocks = 0;
  }
  p.z_blocks = (int)((n_loc + 7) / 8);
  p.x0_blocks = (int)((n_loc + 255) / 256 < 4 * num_sms ? (n_loc + 255) / 256 : 4 * num_sms);
  if (p.x0_blocks < 1) p.x0_blocks = 1;
  p.num_sms = num_sms;
  (void)k;
  return p;
}

cudaError_t est_x0(uint64_t seed, int64_t col0, int64_t n_loc, double2* x, double* part,
                   const EstPlan& p, cudaStream_t st) {
  k_x0<<<p.x0_blocks, 256, 0, st>>>(seed, col0, n_loc, x, part);
  return cudaGetLastError();
}
cudaError_t est_merge_scalar(const double* part, int nparts, double* out, cudaStream_t st) {
  k_merge_scalar<<<1, 256, 0, st>>>(part, nparts, out);
  return cudaGetLastError();
}
cudaError_t est_normalise(const double2* v, int64_t n_loc, const double* nn, double2* x,
                          double* est_out, unsigned long long* vmax, cudaStream_t st) {
  if (vmax) {
    cudaError_t e = cudaMemsetAsync(vmax, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
  }
  int64_t b = (n_loc + 255) / 256;
  if (b > 4096) b = 4096;
  if (b < 1) b = 1;
  k_normalise<<<(unsigned)b, 256, 0, st>>>(v, n_loc, nn, x, est_out, vmax);
  return cudaGetLastError();
}
cudaError_t est_px(const double2* P, int64_t ldp, int64_t k, int64_t n_loc, const double2* x,
                   double* part, double* u_out, const EstPlan& p, cudaStream_t st) {
  k_px<<<p.px_parts, 256, 0, st>>>(P, ldp, k, n_loc, x, p.px_chunk, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_merge_vec_warp<<<(unsigned)((k + 7) / 8), 256, 0, st>>>(part, p.px_parts, k, u_out);
  return cudaGetLastError();
}
cudaError_t est_merge_vec(const double* part, int nparts, int64_t len, double* out, cudaStream_t st) {
  int64_t b = (len + 255) / 256;
  if (b > 4096) b = 4096;
  k_merge_vec<<<(unsigned)b, 256, 0, st>>>(part, nparts, len, out);
  return cudaGetLastError();
}
cudaError_t est_ax(const double2* A, int64_t lda, int64_t m, int64_t n_loc, const double2* x,
                   unsigned long long* bounds, double* part, const EstPlan& p, cudaStream_t st,
                   bool first) {
  if (p.tma) {
    CUtensorMap mapA, mapX;
    cudaError_t e = est_maps(A, lda, m, n_loc, x, n_loc, 16, &mapA, &mapX);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)kEstNS * (kEstBoxA + 128);
    if ((e = ensure_dyn_smem((const void*)k_ax_tma<true>, smem)) != cudaSuccess ||
        (e = ensure_dyn_smem((const void*)k_ax_tma<false>, smem)) != cudaSuccess)
      return e;
    const int nitems = p.ax_rblocks * p.ax_parts;
    const int grid = nitems < 2 * p.num_sms ? nitems : 2 * p.num_sms;
    if (first) {  // amax (bounds[0]) is recorded by this pass
      if ((e = cudaMemsetAsync(bounds, 0, sizeof(unsigned long long), st)) != cudaSuccess) return e;
      k_ax_tma<true><<<grid, 256, smem, st>>>(mapA, mapX, m, p.ax_rblocks, nitems,
                                              p.ax_split_cols, n_loc, bounds, part, bounds);
    } else {
      k_ax_tma<false><<<grid, 256, smem, st>>>(mapA, mapX, m, p.ax_rblocks, nitems,
                                               p.ax_split_cols, n_loc, bounds, part, nullptr);
    }
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((m + 255) / 256), (unsigned)p.ax_parts);
  k_ax<<<grid, 256, 0, st>>>(A, lda, m, n_loc, x, p.ax_split_cols, part);
  return cudaGetLastError();
}
cudaError_t est_y(const double* wpart, int nparts, int64_t m, const double2* B, int64_t ldb,
                  int64_t k, const double* u, double2* y, unsigned long long* vmax,
                  cudaStream_t st) {
  if (vmax) {
    cudaError_t e = cudaMemsetAsync(vmax, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
  }
  k_y<<<(unsigned)((m + 31) / 32), 256, 0, st>>>(wpart, nparts, m, B, ldb, k, u, y, vmax);
  return cudaGetLastError();
}
cudaError_t est_bhy(const double2* B, int64_t ldb, int64_t m, int64_t k, const double2* y,
                    double* sb, cudaStream_t st) {
  k_bhy<<<(unsigned)k, 256, 0, st>>>(B, ldb, m, y, sb);
  return cudaGetLastError();
}
cudaError_t est_z(const double2* A, int64_t lda, int64_t m, int64_t n_loc, const double2* y,
                  const double2* P, int64_t ldp, int64_t k, const double* sb, double2* z,
                  const unsigned long long* bounds, double* npart, const EstPlan& p,
                  cudaStream_t st) {
  if (p.tma) {
    CUtensorMap mapA, mapY;
    cudaError_t e = est_maps(A, lda, m, n_loc, y, m, 2 * kEstRows, &mapA, &mapY);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)kEstNS * (kEstBoxA + kEstRows * 16);
    if ((e = ensure_dyn_smem((const void*)k_z_tma, smem)) != cudaSuccess) return e;
    const int nitems = p.z_blocks;
    const int grid = nitems < 2 * p.num_sms ? nitems : 2 * p.num_sms;
    k_z_tma<<<grid, 256, smem, st>>>(mapA, mapY, m, n_loc, nitems, P, ldp, k, sb, z, bounds,
                                     npart);
    return cudaGetLastError();
  }
  k_z<<<p.z_blocks, 256, 0, st>>>(A, lda, m, n_loc, y, P, ldp, k, sb, z, npart);
  return cudaGetLastError();
}

}  // namespace rid
