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
#include "rid_device.cuh"
#include "rid_internal.h"

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
__global__ void k_normalise(const double2* __restrict__ v, int64_t n_loc, const double* __restrict__ nn,
                            double2* __restrict__ x, double* __restrict__ est_out) {
  const double nv = __dsqrt_rn(__dadd_rn(nn[0], nn[1]));
  if (blockIdx.x == 0 && threadIdx.x == 0 && est_out) est_out[0] = __dsqrt_rn(nv);
  if (!(nv > 0.0)) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_loc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = v[j];
    x[j] = make_double2(__ddiv_rn(a.x, nv), __ddiv_rn(a.y, nv));
  }
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
__global__ void k_y(const double* __restrict__ wpart, int nparts, int64_t m,
                    const double2* __restrict__ B, int64_t ldb, int64_t k,
                    const double* __restrict__ u, double2* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    cdd a = cdd_load(wpart + (size_t)i * 4);
    for (int q = 1; q < nparts; ++q) cdd_merge(a, cdd_load(wpart + ((size_t)q * m + i) * 4));
    for (int64_t t = 0; t < k; ++t) {
      const double2 b = B[t * ldb + i];
      const double4 ut = reinterpret_cast<const double4*>(u)[t];
      const double2 nb = make_double2(-b.x, -b.y);
      cdd_mac(a, nb, make_double2(ut.x, ut.z), false);  // exact part of B u_s
      cdd_mac(a, nb, make_double2(ut.y, ut.w), false);  // B u_c
    }
    y[i] = make_double2(dd_val(a.re), dd_val(a.im));
  }
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

// ------------------------------------------------------------------------------ launchers ------
EstPlan est_plan(int64_t m, int64_t n_loc, int64_t k, int num_sms) {
  EstPlan p;
  p.px_chunk = 64;
  p.px_parts = (int)((n_loc + p.px_chunk - 1) / p.px_chunk);
  const int64_t row_blocks = (m + 255) / 256;
  int64_t splits = (8 * num_sms + row_blocks - 1) / row_blocks;
  if (splits < 1) splits = 1;
  if (splits > n_loc) splits = n_loc;
  if (splits > 1024) splits = 1024;
  p.ax_split_cols = (n_loc + splits - 1) / splits;
  p.ax_parts = (int)((n_loc + p.ax_split_cols - 1) / p.ax_split_cols);
  p.z_blocks = (int)((n_loc + 7) / 8);
  p.x0_blocks = (int)((n_loc + 255) / 256 < 4 * num_sms ? (n_loc + 255) / 256 : 4 * num_sms);
  if (p.x0_blocks < 1) p.x0_blocks = 1;
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
                          double* est_out, cudaStream_t st) {
  int64_t b = (n_loc + 255) / 256;
  if (b > 4096) b = 4096;
  if (b < 1) b = 1;
  k_normalise<<<(unsigned)b, 256, 0, st>>>(v, n_loc, nn, x, est_out);
  return cudaGetLastError();
}
cudaError_t est_px(const double2* P, int64_t ldp, int64_t k, int64_t n_loc, const double2* x,
                   double* part, double* u_out, const EstPlan& p, cudaStream_t st) {
  k_px<<<p.px_parts, 256, 0, st>>>(P, ldp, k, n_loc, x, p.px_chunk, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_merge_vec<<<(unsigned)((k + 127) / 128), 128, 0, st>>>(part, p.px_parts, k, u_out);
  return cudaGetLastError();
}
cudaError_t est_merge_vec(const double* part, int nparts, int64_t len, double* out, cudaStream_t st) {
  int64_t b = (len + 255) / 256;
  if (b > 4096) b = 4096;
  k_merge_vec<<<(unsigned)b, 256, 0, st>>>(part, nparts, len, out);
  return cudaGetLastError();
}
cudaError_t est_ax(const double2* A, int64_t lda, int64_t m, int64_t n_loc, const double2* x,
                   double* part, const EstPlan& p, cudaStream_t st) {
  dim3 grid((unsigned)((m + 255) / 256), (unsigned)p.ax_parts);
  k_ax<<<grid, 256, 0, st>>>(A, lda, m, n_loc, x, p.ax_split_cols, part);
  return cudaGetLastError();
}
cudaError_t est_y(const double* wpart, int nparts, int64_t m, const double2* B, int64_t ldb,
                  int64_t k, const double* u, double2* y, cudaStream_t st) {
  int64_t b = (m + 255) / 256;
  if (b > 4096) b = 4096;
  k_y<<<(unsigned)b, 256, 0, st>>>(wpart, nparts, m, B, ldb, k, u, y);
  return cudaGetLastError();
}
cudaError_t est_bhy(const double2* B, int64_t ldb, int64_t m, int64_t k, const double2* y,
                    double* sb, cudaStream_t st) {
  k_bhy<<<(unsigned)k, 256, 0, st>>>(B, ldb, m, y, sb);
  return cudaGetLastError();
}
cudaError_t est_z(const double2* A, int64_t lda, int64_t m, int64_t n_loc, const double2* y,
                  const double2* P, int64_t ldp, int64_t k, const double* sb, double2* z,
                  double* npart, const EstPlan& p, cudaStream_t st) {
  k_z<<<p.z_blocks, 256, 0, st>>>(A, lda, m, n_loc, y, P, ldp, k, sb, z, npart);
  return cudaGetLastError();
}

}  // namespace rid
