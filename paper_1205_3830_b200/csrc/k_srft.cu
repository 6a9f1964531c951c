// k_srft.cu — the paper's own randomisation Y = S F D A (§2, Eqs. 4–7; NEXT-1 of
// SURVEY.md §8(f)), on B200: an FFT factorisation whose heavy half runs on the DMMA pipe.
//
// With m = m1 * R (R = 16) and i = i1 + m1 * i2, the sampled DFT rows factor as
//     Y(k, c) = sum_{i1} W_m^{(s_k i1) mod m} * Z_c(i1, s_k mod R),
//     Z_c(i1, r) = sum_{i2 < R} W_R^{r i2} * d(i1 + m1 i2) * A(i1 + m1 i2, c)
// (W_N = e^{-2 pi i / N}; W_m^{s m1 i2} = W_R^{s i2}). So:
//   pass 1 (k_srft_pass1): D-scaling and the R-point DFT along i2, one thread per (i1, c), radix-4
//     x radix-4 in registers, coalesced along i1 — one read of A, one write of Z (HBM-bound);
//   pass 2: for each residue r, the rows k with s_k mod R = r form one small complex GEMM
//     Y_r (l_r x n) = W_r (l_r x m1) . Z^(r) (m1 x n) on the same complex-product kernel as the
//     Gaussian sketch (k_zgemm3m.cu, Gauss's three products; the ordered k_zgemm.cu with
//     RID_SKETCH_4M=1) — 6 (or 8) l m n / R real flops instead of the dense 8 l m n.
// Plan (docs/RNG.md §7): d_i = (cos, sin)(2 pi u1) of Philox (i, 0, s_phase, 0) via the spec'd
// sincos, s_k = x0 & (m - 1) of Philox (k, 0, s_sample, 0); W entries from the same sincos on
// u = ((s_k i1) mod m) / m. Agreement with the oracle's direct ascending sum is to rounding.
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "rid_device.cuh"
#include "rid_internal.h"
#include "rid_tma.cuh"

namespace rid {

constexpr int kSrftR = 16;

__global__ void k_srft_plan(uint64_t seed, uint32_t s_phase, uint32_t s_sample, int64_t m,
                            int64_t l, double2* __restrict__ d, int64_t* __restrict__ samples) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = philox4x32_10(make_uint4((uint32_t)i, 0u, s_phase, 0u), k0, k1);
    d[i] = rid_cossin2pi(u01_from(x.x, x.y));
    if (i < l) {
      const uint4 y = philox4x32_10(make_uint4((uint32_t)i, 0u, s_sample, 0u), k0, k1);
      samples[i] = (int64_t)(y.x & (uint32_t)(m - 1));
    }
  }
  // l may exceed m (sampling with replacement)
  for (int64_t i = m + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < l;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 y = philox4x32_10(make_uint4((uint32_t)i, 0u, s_sample, 0u), k0, k1);
    samples[i] = (int64_t)(y.x & (uint32_t)(m - 1));
  }
}

// Stable counting sort of the samples by residue s mod R (one CTA): order[pos] = k, offs[r].
__global__ void k_srft_group(const int64_t* __restrict__ samples, int64_t l, int* __restrict__ order,
                             int* __restrict__ offs) {
  __shared__ int cnt[kSrftR + 1];
  if (threadIdx.x <= kSrftR) cnt[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t k = 0; k < l; ++k) cnt[(int)(samples[k] % kSrftR) + 1]++;
    for (int r = 0; r < kSrftR; ++r) cnt[r + 1] += cnt[r];
    for (int r = 0; r <= kSrftR; ++r) offs[r] = cnt[r];
    for (int64_t k = 0; k < l; ++k) order[cnt[(int)(samples[k] % kSrftR)]++] = (int)k;
  }
}

// Wg(k', i1) = W_m^{(s_{order[k']} i1) mod m}, column-major l x m1 (ld = l)
__global__ void k_srft_wgen(const int64_t* __restrict__ samples, const int* __restrict__ order,
                            int64_t l, int64_t m, int64_t m1, double2* __restrict__ Wg) {
  const int64_t total = l * m1;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kk = q % l, i1 = q / l;
    const uint64_t t = ((uint64_t)samples[order[kk]] * (uint64_t)i1) & (uint64_t)(m - 1);
    const double2 cs = rid_cossin2pi(__ddiv_rn((double)t, (double)m));  // exact: m = 2^p
    Wg[q] = make_double2(cs.x, -cs.y);
  }
}

// Ws(prow(k'), i1) = Re Wg(k', i1) + Im Wg(k', i1) with each residue group starting on an even
// row (ps[r] = sum of the earlier groups' sizes rounded up to even; pad rows zero): the 3M
// kernel's non-swizzled TMA boxes of the plane must start on a 16-byte boundary.
__global__ void k_srft_wsum(const double2* __restrict__ Wg, int64_t l, int64_t m1,
                            const int* __restrict__ offs, double* __restrict__ Ws, int64_t ldws) {
  __shared__ int so[kSrftR + 1], sp[kSrftR + 1];
  if (threadIdx.x == 0) {
    sp[0] = 0;
    for (int r = 0; r <= kSrftR; ++r) so[r] = offs[r];
    for (int r = 0; r < kSrftR; ++r) sp[r + 1] = sp[r] + ((so[r + 1] - so[r] + 1) & ~1);
  }
  __syncthreads();
  const int64_t total = ldws * m1;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i1 = q / ldws, pr = q % ldws;
    int r = 0;
    while (r < kSrftR - 1 && pr >= sp[r + 1]) ++r;
    const int64_t kk = so[r] + (pr - sp[r]);
    double v = 0.0;
    if (pr < sp[kSrftR] && kk < so[r + 1]) {
      const double2 w = Wg[i1 * l + kk];
      v = __dadd_rn(w.x, w.y);
    }
    Ws[q] = v;
  }
}

// complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // * (-i)

// 4-point DFT (forward): X_q = sum_p x_p W_4^{pq}
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), e = mul_mi(csub(x1, x3));
  x0 = cadd(a, c);
  x2 = csub(a, c);
  x1 = cadd(b, e);
  x3 = csub(b, e);
}

__global__ void __launch_bounds__(128) k_srft_pass1(const double2* __restrict__ A, int64_t lda,
                                                    int64_t m1, int64_t n_loc,
                                                    const double2* __restrict__ d,
                                                    double2* __restrict__ Z) {
  // W_16^e, e = 0..9 (the twiddles of the 4 x 4 split: W_16^{p q}, p, q < 4)
  const double c1 = 0.92387953251128674, s1 = 0.38268343236508978, h = 0.70710678118654757;
  const double2 W[10] = {make_double2(1, 0),   make_double2(c1, -s1), make_double2(h, -h),
                         make_double2(s1, -c1), make_double2(0, -1),  make_double2(-s1, -c1),
                         make_double2(-h, -h),  make_double2(-c1, -s1), make_double2(-1, 0),
                         make_double2(-c1, s1)};
  const int64_t i1 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (i1 >= m1) return;
  const double2* a = A + c * lda + i1;
  double2 x[16];
#pragma unroll
  for (int i2 = 0; i2 < 16; ++i2) x[i2] = cmul(__ldg(d + i1 + m1 * i2), __ldcs(a + m1 * i2));
  // 16 = 4 x 4, i2 = p + 4 q: first DFT-4 over q (stride 4) for each p, twiddle W_16^{p r1},
  // then DFT-4 over p; output index r = r1 + 4 r2.
#pragma unroll
  for (int p = 0; p < 4; ++p) dft4(x[p], x[p + 4], x[p + 8], x[p + 12]);  // x[p + 4 r1]
#pragma unroll
  for (int p = 1; p < 4; ++p)
#pragma unroll
    for (int r1 = 1; r1 < 4; ++r1) x[p + 4 * r1] = cmul(x[p + 4 * r1], W[p * r1]);
#pragma unroll
  for (int r1 = 0; r1 < 4; ++r1) dft4(x[4 * r1], x[4 * r1 + 1], x[4 * r1 + 2], x[4 * r1 + 3]);
  // x[4 r1 + r2] now holds output r = r1 + 4 r2
#pragma unroll
  for (int r1 = 0; r1 < 4; ++r1)
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) {
      const int r = r1 + 4 * r2;
      Z[((int64_t)r * n_loc + c) * m1 + i1] = x[4 * r1 + r2];
    }
}

// =============================================================================================
// Single-pass SRFT (default for m >= 2048; SURVEY.md §8(f) NEXT-1's "one HBM pass" model).
// With m = m1 * 256 and i = i1 + m1 * i2:
//     Y(k, c) = sum_{i1 < m1} W_m^{(s_k i1) mod m} * Z_c(i1, s_k mod 256),
//     Z_c(i1, r) = sum_{i2 < 256} W_256^{r i2} * d(i1 + m1 i2) * A(i1 + m1 i2, c).
// One CTA per SM walks column PAIRS; for each pair it streams A in chunks of 8 consecutive i1 x
// all 256 i2 (one 3D TMA box of 32 KB per column, rows 8 KB apart) plus the matching box of the
// phases d, computes the 16 = 2 x 8 DFTs of 256 points in shared memory (radix 16 x 16: pass A
// over i2 = p + 16 q with the W_256^{p r1} twiddle, pass B over p), and accumulates every sampled
// row Y(k, c) += W_m^{s_k i1} Z_c(i1, s_k mod 256) over the chunk's 8 i1 in registers (W_m^{s_k
// i1} = W_m^{(8 q s_k) mod m} from the spec'd sincos, times W_m^{s_k} repeatedly). A is read once
// from HBM; Z never leaves shared memory. Agreement with the oracle's direct ascending sum is to
// rounding (the FFT's log m rounding steps).
// =============================================================================================
constexpr int kSfR = 256;            // first-level DFT length
constexpr int kSfC = 8;              // i1 per chunk
constexpr int kSfBox = kSfR * kSfC * 16;       // bytes: one column's (or d's) chunk, 32 KB
constexpr int kSfStage = 3 * kSfBox;           // A of two columns + d
// NS stages per CTA, NB CTAs per SM: (2, 1) double-buffers one CTA; (1, 2) runs two
// single-buffered CTAs per SM that hide each other's loads (twice the warps)
template <int NS>
constexpr size_t sf_smem() {
  return (size_t)NS * kSfStage + kSfR * 16 + 1024;
}

// 16-point DFT in registers (4 x 4; the pass-1 kernel's scheme): x[p] in, x[4 r1 + r2] = X(r1 + 4 r2)
__device__ __forceinline__ void dft16(double2 (&x)[16]) {
  const double c1 = 0.92387953251128674, s1 = 0.38268343236508978, h = 0.70710678118654757;
  const double2 W[10] = {make_double2(1, 0),   make_double2(c1, -s1), make_double2(h, -h),
                         make_double2(s1, -c1), make_double2(0, -1),  make_double2(-s1, -c1),
                         make_double2(-h, -h),  make_double2(-c1, -s1), make_double2(-1, 0),
                         make_double2(-c1, s1)};
#pragma unroll
  for (int p = 0; p < 4; ++p) dft4(x[p], x[p + 4], x[p + 8], x[p + 12]);
#pragma unroll
  for (int p = 1; p < 4; ++p)
#pragma unroll
    for (int r1 = 1; r1 < 4; ++r1) x[p + 4 * r1] = cmul(x[p + 4 * r1], W[p * r1]);
#pragma unroll
  for (int r1 = 0; r1 < 4; ++r1) dft4(x[4 * r1], x[4 * r1 + 1], x[4 * r1 + 2], x[4 * r1 + 3]);
}

__device__ __forceinline__ void tma_box3_g2s(void* dst, const CUtensorMap* map, int x, int y, int z,
                                             uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(b))
      : "memory");
}

// KPT: sampled rows per thread (l <= 256 KPT). Pairs (2c, 2c + 1) of the n_loc columns (an odd
// last column is paired with itself and written once).
template <int KPT, int kSfStages, int NB>
__global__ void __launch_bounds__(256, NB)
    k_srft_fused(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapD,
                 int64_t m, int64_t m1, int64_t n_loc, int64_t l,
                 const int64_t* __restrict__ samples, double2* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(1024) unsigned char sfraw[];
  __shared__ __align__(8) uint64_t full[kSfStages];
  unsigned char* sm = sfraw + ((1024 - (smem_u32(sfraw) & 1023)) & 1023);
  double2* tw256 = reinterpret_cast<double2*>(sm + (size_t)kSfStages * kSfStage);  // W_256^e
  const int tid = threadIdx.x;
  const int64_t npairs = (n_loc + 1) / 2;
  const int nq = (int)(m1 / kSfC);  // chunks per column pair
  // this CTA's items: (pair, chunk) for its pairs b, b + G, ...
  const int64_t mypairs = (npairs > blockIdx.x) ? (npairs - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nitems = mypairs * nq;

  for (int e = tid; e < kSfR; e += blockDim.x) {  // W_256^e = (cos, -sin)(2 pi e / 256)
    const double2 cs = rid_cossin2pi(__ddiv_rn((double)e, 256.0));
    tw256[e] = make_double2(cs.x, -cs.y);
  }
  if (tid == 0) {
    tma_prefetch_map(&mapA);
    tma_prefetch_map(&mapD);
    for (int s = 0; s < kSfStages; ++s) mbar_init(&full[s], 1);
    mbar_init_fence();
  }
  __syncthreads();

  auto issue = [&](int64_t it) {  // thread 0
    const int s = (int)(it % kSfStages);
    const int64_t pr = blockIdx.x + (it / nq) * (int64_t)gridDim.x;
    const int q = (int)(it % nq);
    const int64_t c0 = 2 * pr, c1 = (2 * pr + 1 < n_loc) ? 2 * pr + 1 : 2 * pr;
    unsigned char* st = sm + (size_t)s * kSfStage;
    mbar_expect_tx(&full[s], kSfStage);
    tma_box3_g2s(st, &mapA, 2 * kSfC * q, 0, (int)c0, &full[s]);
    tma_box3_g2s(st + kSfBox, &mapA, 2 * kSfC * q, 0, (int)c1, &full[s]);
    tma_box3_g2s(st + 2 * kSfBox, &mapD, 2 * kSfC * q, 0, 0, &full[s]);
  };
  if (tid == 0)
    for (int64_t it = 0; it < kSfStages && it < nitems; ++it) issue(it);

  // owned samples k = tid + 256 j: s_k, W_m^{s_k}, and W_m^{s_k rot}: a lane reads the chunk's 8
  // i1 of Z starting at c = rot = tid & 7 (the 8 lanes of a shared-memory wavefront then hit 8
  // different bank groups), so its twiddle starts at W_m^{s_k (8 q + rot)}
  const int rot = tid & 7;
  const double inv_m = __drcp_rn((double)m);  // m = 2^p: exact
  int64_t sk[KPT];
  double2 step[KPT], steprot[KPT];
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int64_t k = tid + 256 * j;
    sk[j] = k < l ? samples[k] : 0;
    const double2 cs = rid_cossin2pi(__ddiv_rn((double)sk[j], (double)m));
    step[j] = make_double2(cs.x, -cs.y);
    const uint64_t tr = ((uint64_t)sk[j] * (uint64_t)rot) & (uint64_t)(m - 1);
    const double2 cr = rid_cossin2pi(__ddiv_rn((double)tr, (double)m));
    steprot[j] = make_double2(cr.x, -cr.y);
  }
  double2 acc[2][KPT];
#pragma unroll
  for (int j = 0; j < KPT; ++j) acc[0][j] = acc[1][j] = make_double2(0.0, 0.0);

  // pass roles: thread -> (column cc, i1c, p) for pass A and (cc, i1c, r1) for pass B, i1c fastest:
  // a row of the box holds the 8 i1 of one i2, so the 8 lanes of a wavefront hit 8 bank groups
  const int cc = tid >> 7, i1c = tid & 7, pp = (tid >> 3) & 15;
  for (int64_t it = 0; it < nitems; ++it) {
    const int s = (int)(it % kSfStages);
    const int q = (int)(it % nq);
    mbar_wait(&full[s], (unsigned)((it / kSfStages) & 1));
    double2* Zc = reinterpret_cast<double2*>(sm + (size_t)s * kSfStage + (size_t)cc * kSfBox);
    const double2* Dd = reinterpret_cast<const double2*>(sm + (size_t)s * kSfStage + 2 * kSfBox);
    // ---- pass A: x(pp + 16 q2) d(.) over q2, DFT-16, twiddle W_256^{pp r1}, in place ---------
    {
      double2 x[16];
#pragma unroll
      for (int q2 = 0; q2 < 16; ++q2) {
        const int i2 = pp + 16 * q2;
        x[q2] = cmul(Dd[i2 * kSfC + i1c], Zc[i2 * kSfC + i1c]);
      }
      dft16(x);  // x[4 a + b] = y(r1 = a + 4 b)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int r1 = a + 4 * b;
          Zc[(pp + 16 * r1) * kSfC + i1c] = cmul(x[4 * a + b], tw256[pp * r1]);
        }
    }
    __syncthreads();
    // ---- pass B: thread (cc, i1c, r1 = pp) reads y(p, r1) for p < 16, DFT-16 over p ----------
    {
      double2 x[16];
#pragma unroll
      for (int p = 0; p < 16; ++p) x[p] = Zc[(p + 16 * pp) * kSfC + i1c];
      dft16(x);  // x[4 a + b] = X(r1 + 16 r2), r2 = a + 4 b
      __syncthreads();  // every read of pass B before any write
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) Zc[(pp + 16 * (a + 4 * b)) * kSfC + i1c] = x[4 * a + b];
    }
    __syncthreads();
    // ---- accumulate the chunk's 8 i1 into every owned sampled row, both columns -------------
    const double2* Z0 = reinterpret_cast<const double2*>(sm + (size_t)s * kSfStage);
    const double2* Z1 = reinterpret_cast<const double2*>(sm + (size_t)s * kSfStage + kSfBox);
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (tid + 256 * j >= l) continue;
      const int r = (int)(sk[j] & (kSfR - 1));
      const uint64_t t0 = ((uint64_t)sk[j] * (uint64_t)(kSfC * q)) & (uint64_t)(m - 1);
      const double2 cs = rid_cossin2pi(__dmul_rn((double)t0, inv_m));  // t0 / m, exact
      const double2 wbase = make_double2(cs.x, -cs.y);  // W_m^{s_k 8 q}
      double2 w = cmul(wbase, steprot[j]);              // W_m^{s_k (8 q + rot)}
#pragma unroll
      for (int i = 0; i < kSfC; ++i) {
        const int c = (i + rot) & (kSfC - 1);  // i1 = 8 q + c
        if (c == 0 && i > 0) w = wbase;        // wrapped past c = 7
        const double2 z0 = Z0[r * kSfC + c], z1 = Z1[r * kSfC + c];
        acc[0][j].x = __fma_rn(w.x, z0.x, __fma_rn(-w.y, z0.y, acc[0][j].x));
        acc[0][j].y = __fma_rn(w.x, z0.y, __fma_rn(w.y, z0.x, acc[0][j].y));
        acc[1][j].x = __fma_rn(w.x, z1.x, __fma_rn(-w.y, z1.y, acc[1][j].x));
        acc[1][j].y = __fma_rn(w.x, z1.y, __fma_rn(w.y, z1.x, acc[1][j].y));
        w = cmul(w, step[j]);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();  // stage s consumed by every thread
    if (tid == 0 && it + kSfStages < nitems) issue(it + kSfStages);
    if (q == nq - 1) {  // the pair is complete
      const int64_t pr = blockIdx.x + (it / nq) * (int64_t)gridDim.x;
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int64_t k = tid + 256 * j;
        if (k < l) {
          Y[(2 * pr) * ldy + k] = acc[0][j];
          if (2 * pr + 1 < n_loc) Y[(2 * pr + 1) * ldy + k] = acc[1][j];
        }
        acc[0][j] = acc[1][j] = make_double2(0.0, 0.0);
      }
    }
  }
}

bool srft_fused_enabled(int64_t m, int64_t l) {
  const char* v = select_env("RID_SRFT_FUSED");  // 0: the two-pass SRFT (DFT-16 + DMMA products)
  return !(v && atoi(v) == 0) && m >= (int64_t)kSfR * kSfC && l <= 2048;
}

static cudaError_t srft_fused(uint64_t seed, bool retry, int64_t l, const double2* A, int64_t m,
                              int64_t n_loc, int64_t lda, double2* Y, int64_t ldy, void* work,
                              int num_sms, cudaStream_t st, int* launches) {
  const int64_t m1 = m / kSfR;
  char* w = (char*)work;
  double2* d = (double2*)w;
  int64_t* samples = (int64_t*)(w + (((size_t)m * sizeof(double2) + 255) & ~(size_t)255));
  const uint32_t sp = retry ? 22u : 6u, ss = retry ? 23u : 7u;
  int64_t blocks = ((m > l ? m : l) + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_srft_plan<<<(unsigned)blocks, 256, 0, st>>>(seed, sp, ss, m, l, d, samples);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  *launches += 1;
  PFN_cuTensorMapEncodeTiled encode;
  if ((e = tensor_map_encoder(&encode)) != cudaSuccess) return e;
  // A as (2 m1 doubles: i1) x 256 (i2, m1 complex apart) x n_loc (columns); d the same, 1 column
  CUtensorMap mapA, mapD;
  const cuuint32_t box[3] = {(cuuint32_t)(2 * kSfC), (cuuint32_t)kSfR, 1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  {
    const cuuint64_t gdim[3] = {(cuuint64_t)(2 * m1), (cuuint64_t)kSfR, (cuuint64_t)n_loc};
    const cuuint64_t gstr[2] = {(cuuint64_t)m1 * sizeof(double2), (cuuint64_t)lda * sizeof(double2)};
    if (encode(&mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)A, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t gdim[3] = {(cuuint64_t)(2 * m1), (cuuint64_t)kSfR, 1u};
    const cuuint64_t gstr[2] = {(cuuint64_t)m1 * sizeof(double2), (cuuint64_t)m * sizeof(double2)};
    if (encode(&mapD, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)d, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int64_t npairs = (n_loc + 1) / 2;
  // 1: two single-buffered CTAs per SM (128 registers: l <= 512 fits without spills); 0: one
  // double-buffered CTA per SM
  int cfg = l <= 512 ? 1 : 0;
  if (const char* v = experiment_env("RID_SRFT_CFG")) cfg = atoi(v);
  const int64_t slots = (int64_t)num_sms * (cfg ? 2 : 1);
  const unsigned grid = (unsigned)(npairs < slots ? npairs : slots);
#define RID_SF(K)                                                                              \
  {                                                                                            \
    if (cfg) {                                                                                 \
      auto kern = k_srft_fused<K, 1, 2>;                                                       \
      if ((e = ensure_dyn_smem((const void*)kern, sf_smem<1>())) != cudaSuccess) return e;     \
      kern<<<grid, 256, sf_smem<1>(), st>>>(mapA, mapD, m, m1, n_loc, l, samples, Y, ldy);     \
    } else {                                                                                   \
      auto kern = k_srft_fused<K, 2, 1>;                                                       \
      if ((e = ensure_dyn_smem((const void*)kern, sf_smem<2>())) != cudaSuccess) return e;     \
      kern<<<grid, 256, sf_smem<2>(), st>>>(mapA, mapD, m, m1, n_loc, l, samples, Y, ldy);     \
    }                                                                                          \
    *launches += 1;                                                                            \
    return cudaGetLastError();                                                                 \
  }
  if (l <= 256) RID_SF(1)
  if (l <= 512) RID_SF(2)
  if (l <= 1024) RID_SF(4)
  RID_SF(8)
#undef RID_SF
}

__global__ void k_srft_scatter(const double2* __restrict__ Yg, const int* __restrict__ order,
                               int64_t l, int64_t n_loc, double2* __restrict__ Y, int64_t ldy) {
  const int64_t total = l * n_loc;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kk = q % l, c = q / l;
    Y[c * ldy + order[kk]] = Yg[q];
  }
}

// Column chunk of the two passes: Z is as large as A's chunk, so a chunk of ~4 GiB of A bounds
// the workspace (C5: 2048 columns per chunk) while every GEMM still has >= 2 CTAs per SM.
int64_t srft_chunk_cols(int64_t m, int64_t n_loc) {
  int64_t c = ((int64_t)4 << 30) / (16 * m);
  if (c < 64) c = 64;
  return c < n_loc ? c : n_loc;
}

size_t srft_work_bytes(int64_t m, int64_t l, int64_t n_loc) {
  const int64_t m1 = m / kSrftR, ch = srft_chunk_cols(m, n_loc);
  return sizeof(double2) * ((size_t)m + (size_t)l * m1 + (size_t)kSrftR * m1 * ch +
                            (size_t)l * ch) +
         sizeof(double) * (size_t)(rsum_ld(l) + kSrftR) * m1 +  // Re Wg + Im Wg, padded
         sizeof(int64_t) * (size_t)l + sizeof(int) * ((size_t)l + kSrftR + 1) + 2304;
}

cudaError_t srft_sketch(uint64_t seed, bool retry, int64_t l, const double2* A, int64_t m,
                        int64_t n, int64_t n_loc, int64_t lda, double2* Y, int64_t ldy, void* work,
                        double2* splitk, size_t splitk_elems, int num_sms, cudaStream_t st,
                        int* launches) {
  if (m < kSrftR || (m & (m - 1)) != 0) return cudaErrorInvalidValue;
  if (srft_fused_enabled(m, l))
    return srft_fused(seed, retry, l, A, m, n_loc, lda, Y, ldy, work, num_sms, st, launches);
  const int64_t m1 = m / kSrftR, ch = srft_chunk_cols(m, n_loc);
  if (ch > 65535) return cudaErrorInvalidConfiguration;
  char* w = (char*)work;
  auto take = [&](size_t bytes) {
    char* p = w;
    w += (bytes + 255) & ~(size_t)255;
    return (void*)p;
  };
  double2* d = (double2*)take(sizeof(double2) * m);
  double2* Wg = (double2*)take(sizeof(double2) * l * m1);
  const int64_t ldws = rsum_ld(l) + kSrftR;  // >= every padded group layout, even
  double* Wgs = (double*)take(sizeof(double) * ldws * m1);  // Re Wg + Im Wg (3M sums)
  double2* Z = (double2*)take(sizeof(double2) * kSrftR * m1 * ch);
  double2* Yg = (double2*)take(sizeof(double2) * l * ch);
  int64_t* samples = (int64_t*)take(sizeof(int64_t) * l);
  int* order = (int*)take(sizeof(int) * l);
  int* offs = (int*)take(sizeof(int) * (kSrftR + 1));
  const uint32_t sp = retry ? 22u : 6u, ss = retry ? 23u : 7u;
  int64_t blocks = ((m > l ? m : l) + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_srft_plan<<<(unsigned)blocks, 256, 0, st>>>(seed, sp, ss, m, l, d, samples);
  k_srft_group<<<1, 32, 0, st>>>(samples, l, order, offs);
  int64_t wb = (l * m1 + 255) / 256;
  if (wb > 8192) wb = 8192;
  k_srft_wgen<<<(unsigned)wb, 256, 0, st>>>(samples, order, l, m, m1, Wg);
  {
    int64_t sb = (ldws * m1 + 255) / 256;
    if (sb > 8192) sb = 8192;
    k_srft_wsum<<<(unsigned)sb, 256, 0, st>>>(Wg, l, m1, offs, Wgs, ldws);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int hoffs[kSrftR + 1];
  e = cudaMemcpyAsync(hoffs, offs, sizeof(hoffs), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  *launches += 4;
  for (int64_t c0 = 0; c0 < n_loc; c0 += ch) {
    const int64_t nc = (c0 + ch <= n_loc) ? ch : n_loc - c0;
    dim3 g1((unsigned)((m1 + 127) / 128), (unsigned)nc);
    k_srft_pass1<<<g1, 128, 0, st>>>(A + c0 * lda, lda, m1, nc, d, Z);
    *launches += 1;
    if (sketch_mults() == 3) {  // the 16 residue products in one batched launch (no K split)
      Z3Batch bt{};
      for (int r = 0; r < kSrftR; ++r) {
        const int64_t lr = hoffs[r + 1] - hoffs[r];
        if (lr == 0) continue;
        bt.roff[bt.n] = hoffs[r];
        bt.boff[bt.n] = (int64_t)r * m1 * nc;
        bt.coff[bt.n] = hoffs[r];
        bt.mout[bt.n] = lr;
        ++bt.n;
      }
      const char* v = select_env("RID_Z3_TMA");
      if (v && atoi(v) == 0) {
        e = zgemm3m_batched(Wg, l, Z, m1, Yg, l, bt, nc, m1, st);
        if (e != cudaSuccess) return e;
        *launches += 1;
      } else {
        // each residue's l_r rows cut into 48-, 40- and 24-row tiles with the fewest padded rows
        // (l_r ~ l/16 ± 25%: one fixed height pads 20-30% of the residue products), one batched
        // launch per tile height
        Z3Batch bh[3] = {};
        const int hts[3] = {48, 40, 24};
        int64_t ps[kSrftR + 1];  // even-padded group starts in Wgs (k_srft_wsum)
        ps[0] = 0;
        for (int r = 0; r < kSrftR; ++r) ps[r + 1] = ps[r] + ((hoffs[r + 1] - hoffs[r] + 1) & ~1);
        int zr[kZ3BatchMax];  // residue of item z of bt
        for (int r = 0, z = 0; r < kSrftR; ++r)
          if (hoffs[r + 1] > hoffs[r]) zr[z++] = r;
        for (int z = 0; z < bt.n; ++z) {
          const int64_t lr = bt.mout[z];
          int64_t best = INT64_MAX;
          int cnt[3] = {0, 0, 0};
          for (int a3 = 0; a3 <= (int)((lr + 47) / 48); ++a3)
            for (int b3 = 0; b3 <= 2; ++b3)
              for (int c3 = 0; c3 <= 2; ++c3) {
                const int64_t cover = 48 * a3 + 40 * b3 + 24 * c3;
                if (cover < lr) continue;
                const int64_t cost = (cover - lr) * 16 + a3 + b3 + c3;  // padding, then tiles
                if (cost < best) {
                  best = cost;
                  cnt[0] = a3;
                  cnt[1] = b3;
                  cnt[2] = c3;
                }
              }
          int64_t row = 0;
          for (int h = 0; h < 3 && row < lr; ++h) {
            if (cnt[h] == 0) continue;
            const int64_t rows = (lr - row < (int64_t)cnt[h] * hts[h]) ? lr - row : (int64_t)cnt[h] * hts[h];
            Z3Batch& q = bh[h];
            q.roff[q.n] = bt.roff[z] + row;
            q.soff[q.n] = ps[zr[z]] + row;  // row is a multiple of 48 / 40 / 24: even
            q.boff[q.n] = bt.boff[z];
            q.coff[q.n] = bt.coff[z] + row;
            q.mout[q.n] = rows;
            ++q.n;
            row += rows;
          }
        }
        for (int h = 0; h < 3; ++h) {
          if (bh[h].n == 0) continue;
          e = zgemm3m_tma_batched_h(Wg, l, l, Z, m1, kSrftR * nc, Yg, l, bh[h], nc, m1, hts[h], st,
                                    Wgs, ldws, ps[kSrftR]);
          if (e != cudaSuccess) return e;
          *launches += 1;
        }
      }
    } else {
      for (int r = 0; r < kSrftR; ++r) {
        const int64_t lr = hoffs[r + 1] - hoffs[r];
        if (lr == 0) continue;
        int S = zgemm_ksplit(lr, m1, n / 8, num_sms);
        if ((size_t)S * lr * nc > splitk_elems) S = 1;
        e = zgemm_ordered(Wg + hoffs[r], l, Z + (int64_t)r * m1 * nc, m1, Yg + hoffs[r], l, lr,
                          nc, m1, 0, 0.0, 0, 0, st, S, splitk);
        if (e != cudaSuccess) return e;
        *launches += S > 1 ? 2 : 1;
      }
    }
    int64_t sb = (l * nc + 255) / 256;
    if (sb > 8192) sb = 8192;
    k_srft_scatter<<<(unsigned)sb, 256, 0, st>>>(Yg, order, l, nc, Y + c0 * ldy, ldy);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace rid
