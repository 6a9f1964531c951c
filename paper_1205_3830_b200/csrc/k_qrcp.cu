// k_qrcp.cu — column-pivoted Householder QR of the sketch Y (l x n), k steps, one persistent
// cooperative kernel with one grid barrier per step.
//
// Paper: "a highly approximate QR factorization on the matrix Y ... Y ≈ QR" with a column
// permutation "so that the first k columns are linearly independent and contain the k most
// weighted vectors" (§2, Eqs. 8–9); the authors note Householder "should result
// in similar stability with only half the runtime" of their CGS (§3.2).
// Readings: R8 greedy max residual 2-norm pivot, ties -> lowest column index;
// R11 the residual norms are recomputed exactly from the updated column every step (no
// downdating); R13 rank failure when nu_p < 1e-13 * max_c ||Y[:, c]||.
//
// Deferred write-back (the kernel is HBM-bound: one step touches the whole trailing block):
// steps are grouped in blocks of QB. Y is materialised only at block boundaries; inside a block,
// step j = j0 + t reloads each trailing column's block-start segment y^(j0)[j0:l], re-applies the
// t + 1 reflectors H_j0 .. H_j in registers (they sit in shared memory) and recomputes the exact
// residual norm of rows j+1..l-1 from that vector — the same numbers as a step-by-step update,
// but each step reads the trailing block once and writes it only at the end of the block
// (1 + 1/QB passes instead of 2). The FP64 work grows to ≈ 4 (QB + 1) FMA per element per step,
// which the FP64 pipe absorbs (B200: 64 FMA/clk/SM against ≈1.4 elements/clk/SM of HBM).
//
// Work split: every CTA owns a contiguous block of columns. A column's segment is handled by a
// group of `lpc` lanes (32, 16, 8 or 4 — chosen per block so that each lane holds at most MAXQ
// rows in registers): as the trailing block shrinks a warp works on 32/lpc columns at once.
// Every CTA rebuilds the same reflector from column p (identical bits: same code, same data,
// commutative butterfly reductions), so the only cross-CTA exchange is the per-CTA
// (best, second, index) candidate triple.
//
// Output: rows 0..k-1 of every non-pivot column of Y hold R12 (materialised at the last block
// end); the pivot triangle R11 (k x k, column s = pivot step s, diagonal beta real) is written
// densely to out.R11 by CTA 0; out.beta[s] = R11[s, s].
#include <cfloat>
#include <cstdint>

#include "rid_device.cuh"
#include "rid_internal.h"

namespace rid {

struct Top2 {
  double b1;     // best value
  double b2;     // second-best value
  long long i1;  // index of best
};

__device__ __forceinline__ bool beats(double v, long long i, double bv, long long bi) {
  return v > bv || (v == bv && i < bi);
}
__device__ __forceinline__ void top2_init(Top2& a) {
  a.b1 = -1.0;
  a.b2 = -1.0;
  a.i1 = 0x7FFFFFFFFFFFFFFFLL;
}
__device__ __forceinline__ void top2_push(Top2& a, double v, long long i) {
  if (beats(v, i, a.b1, a.i1)) {
    a.b2 = a.b1;
    a.b1 = v;
    a.i1 = i;
  } else if (v > a.b2) {
    a.b2 = v;
  }
}
__device__ __forceinline__ void top2_merge(Top2& a, const Top2& c) {
  if (beats(c.b1, c.i1, a.b1, a.i1)) {
    a.b2 = fmax(a.b1, c.b2);
    a.b1 = c.b1;
    a.i1 = c.i1;
  } else {
    a.b2 = fmax(a.b2, c.b1);
  }
}
__device__ __forceinline__ void top2_warp(Top2& a) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    Top2 o;
    o.b1 = __shfl_xor_sync(0xffffffffu, a.b1, m);
    o.b2 = __shfl_xor_sync(0xffffffffu, a.b2, m);
    o.i1 = __shfl_xor_sync(0xffffffffu, a.i1, m);
    top2_merge(a, o);
  }
}
// butterfly sum over groups of `lpc` lanes (lpc a power of two): every lane of a group ends with
// the same bits (fp addition is commutative)
__device__ __forceinline__ double group_sum(double v, int lpc) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1)
    if (m < lpc) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire(bar) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kQrcpThreads = 256;
constexpr int kQrcpWarps = kQrcpThreads / 32;
// Steps per deferred-write block. Measured on B200 (C4, tools/trace_qrcp.py): QB = 4 cut the
// write traffic but every extra reflector re-read v from shared memory for every column
// (≈27 us per reflector per step at C4: shared-memory bound), so the update pass went from
// 98 to 61/83/110/153 us for t = 0..3. QB = 1 (write every step) is the faster choice until the
// block update moves onto the tensor pipe.
constexpr int kQB = 1;

// lanes per column for a segment of `rows` rows: the smallest group that keeps every lane at
// <= MAXQ rows (more columns per warp as the segment shrinks)
__device__ __forceinline__ int pick_lpc(int rows, int maxq) {
  int lpc = 32;
  while (lpc > 4 && rows <= (lpc / 2) * maxq) lpc >>= 1;
  return lpc;
}

// y <- H^H y for the reflector stored in v (zeros above its pivot row), tau = (tr, ti); every
// lane of the lpc-group holds rows sl + lpc*q of the segment.
template <int MAXQ>
__device__ __forceinline__ void apply_reflector(double2 (&y)[MAXQ], const double2* v, double tr,
                                                double ti, int sl, int lpc, int L) {
  double wr = 0.0, wi = 0.0;
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    const int rr = sl + lpc * q;
    if (rr < L) {
      const double2 vv = v[rr];
      wr = __fma_rn(vv.x, y[q].x, __fma_rn(vv.y, y[q].y, wr));   // conj(v) * y
      wi = __fma_rn(vv.x, y[q].y, __fma_rn(-vv.y, y[q].x, wi));
    }
  }
  wr = group_sum(wr, lpc);
  wi = group_sum(wi, lpc);
  const double s_re = __fma_rn(tr, wr, __dmul_rn(ti, wi));    // s = conj(tau) * w
  const double s_im = __fma_rn(tr, wi, -__dmul_rn(ti, wr));
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    const int rr = sl + lpc * q;
    if (rr < L) {
      const double2 vv = v[rr];
      y[q].x = __fma_rn(-s_re, vv.x, __fma_rn(s_im, vv.y, y[q].x));  // y -= s * v
      y[q].y = __fma_rn(-s_re, vv.y, __fma_rn(-s_im, vv.x, y[q].y));
    }
  }
}

template <int MAXQ>
__global__ void __launch_bounds__(kQrcpThreads, 2)
    k_qrcp(double2* __restrict__ Y, int64_t ldy, int l, int64_t n, int k, double tol_rel,
           QrcpOut out, QrcpWork w) {
  extern __shared__ double2 sv_raw[];  // kQB reflectors of the current block, rows j0..l-1
  double2(*sv)[MAXQ * 32] = reinterpret_cast<double2(*)[MAXQ * 32]>(sv_raw);
  __shared__ double s_tau[kQB][2];
  __shared__ Top2 sred[kQrcpWarps];
  __shared__ long long s_p;
  __shared__ int s_stop;

  const int nb = gridDim.x, b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (n + nb - 1) / nb;
  const int64_t c_lo = (int64_t)b * per;
  const int64_t c_hi = (c_lo + per < n) ? c_lo + per : n;
  double nu0max = 0.0;
  unsigned phase = 0;

  auto block_top2_publish = [&](Top2 loc, int parity) {
    top2_warp(loc);
    if (lane == 0) sred[warp] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
      Top2 t = sred[0];
      for (int q = 1; q < kQrcpWarps; ++q) top2_merge(t, sred[q]);
      double* c = w.cand + ((size_t)parity * w.max_blocks + b) * 3;
      c[0] = t.b1;
      c[1] = t.b2;
      c[2] = (double)t.i1;
    }
  };

  // ---- phase 0: initial column norms --------------------------------------------------------
  {
    const int lpc = pick_lpc(l, MAXQ);
    const int cpw = 32 / lpc, sg = lane / lpc, sl = lane % lpc;
    Top2 loc;
    top2_init(loc);
    for (int64_t c0 = c_lo + (int64_t)warp * cpw; c0 < c_hi; c0 += (int64_t)kQrcpWarps * cpw) {
      const int64_t c = c0 + sg;
      const bool live = c < c_hi;
      const double2* yc = Y + c * ldy;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int r = sl + lpc * q;
        if (live && r < l) {
          const double2 y = yc[r];
          s = __fma_rn(y.x, y.x, s);
          s = __fma_rn(y.y, y.y, s);
        }
      }
      const double nu = __dsqrt_rn(group_sum(s, lpc));
      if (live && sl == 0) {
        w.nu[c] = nu;
        top2_push(loc, nu, c);  // one lane per column: the multiset of candidates has no copies
      }
    }
    block_top2_publish(loc, 0);
    grid_barrier(w.bar, (unsigned)nb * (++phase));
  }

  for (int j = 0; j < k; ++j) {
    const int j0 = j - j % kQB;  // block start
    const int t = j - j0;        // position in the block
    const int L = l - j0;        // segment length (rows j0..l-1)
    const bool block_end = (t == kQB - 1) || (j == k - 1);
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[4 * j + 0] = globaltimer();
    // ---- 1. global pivot: reduce the per-CTA candidates (every CTA, identically) ------------
    if (warp == 0) {
      Top2 tt;
      top2_init(tt);
      const double* cb = w.cand + (size_t)(j & 1) * w.max_blocks * 3;
      for (int q = lane; q < nb; q += 32) {
        Top2 o;
        o.b1 = cb[q * 3 + 0];
        o.b2 = cb[q * 3 + 1];
        o.i1 = (long long)cb[q * 3 + 2];
        top2_merge(tt, o);
      }
      top2_warp(tt);
      if (j == 0) nu0max = tt.b1;  // max_c ||Y[:, c]||
      if (lane == 0) {
        s_p = tt.i1;
        s_stop = (!(tt.b1 >= tol_rel * nu0max) || tt.b1 <= 0.0) ? 1 : 0;
        if (b == 0) {
          out.resid[j] = tt.b1;
          out.margin[j] = (tt.b2 < 0.0) ? DBL_MAX : (tt.b1 - tt.b2) / tt.b1;
          if (!s_stop) out.J[j] = tt.i1;
        }
      }
    }
    __syncthreads();
    if (s_stop) {
      if (b == 0 && threadIdx.x == 0) {
        out.info[0] = 2;
        out.info[1] = j;
      }
      return;  // every CTA takes the same decision at the same step
    }
    const int64_t p = s_p;

    // ---- 2. reflector H_j from x = (H_{j-1} .. H_j0)^H y_p^(j0) rows j..l-1 (zlarfg) ---------
    if (warp == 0) {
      const double2* yp = Y + p * ldy + j0;
      double2 x[MAXQ];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int rr = lane + 32 * q;
        x[q] = (rr < L) ? yp[rr] : make_double2(0.0, 0.0);
      }
      for (int i = 0; i < t; ++i) apply_reflector<MAXQ>(x, sv[i], s_tau[i][0], s_tau[i][1], lane, 32, L);
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int rr = lane + 32 * q;
        if (rr > t && rr < L) {
          s = __fma_rn(x[q].x, x[q].x, s);
          s = __fma_rn(x[q].y, x[q].y, s);
        }
      }
      const double xnorm2 = group_sum(s, 32);
      // alpha = x at row j (relative row t): held by lane t % 32, slot t / 32
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q)
        if (q == t / 32) {
          ar = x[q].x;
          ai = x[q].y;
        }
      ar = __shfl_sync(0xffffffffu, ar, t % 32);
      ai = __shfl_sync(0xffffffffu, ai, t % 32);
      double tau_re, tau_im, beta, sc_re, sc_im;
      if (xnorm2 == 0.0 && ai == 0.0) {
        tau_re = 0.0;
        tau_im = 0.0;
        beta = ar;
        sc_re = 0.0;
        sc_im = 0.0;
      } else {
        const double nrm = __dsqrt_rn(__fma_rn(ar, ar, __fma_rn(ai, ai, xnorm2)));
        beta = (ar >= 0.0) ? -nrm : nrm;
        tau_re = __ddiv_rn(__dsub_rn(beta, ar), beta);
        tau_im = __ddiv_rn(-ai, beta);
        const double dr = __dsub_rn(ar, beta), di = ai;  // scal = 1 / (alpha - beta)
        const double den = __fma_rn(dr, dr, __dmul_rn(di, di));
        sc_re = __ddiv_rn(dr, den);
        sc_im = __ddiv_rn(-di, den);
      }
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int rr = lane + 32 * q;
        if (rr < L) {
          double2 v;
          if (rr < t) {
            v = make_double2(0.0, 0.0);
          } else if (rr == t) {
            v = make_double2(1.0, 0.0);
          } else {
            v.x = __fma_rn(x[q].x, sc_re, -__dmul_rn(x[q].y, sc_im));
            v.y = __fma_rn(x[q].x, sc_im, __dmul_rn(x[q].y, sc_re));
          }
          sv[t][rr] = v;
          // pivot column of R11: rows j0..j-1 are the transformed x, rows < j0 are final in Y
          if (b == 0 && rr < t) out.R11[(int64_t)j * k + j0 + rr] = x[q];
        }
      }
      if (lane == 0) {
        s_tau[t][0] = tau_re;
        s_tau[t][1] = tau_im;
        if (b == 0) {
          out.beta[j] = beta;
          out.R11[(int64_t)j * k + j] = make_double2(beta, 0.0);
        }
      }
    }
    __syncthreads();
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[4 * j + 1] = globaltimer();

    // ---- 3. every owned trailing column: reload y^(j0), apply H_j0..H_j, exact norm ----------
    // rows 0..j0-1 of the pivot column are final (nobody writes them again): CTA 0's last warp
    // copies them into the dense R11 off the critical path (R11 is zeroed before the launch)
    if (b == 0 && warp == kQrcpWarps - 1)
      for (int r = lane; r < j0; r += 32) out.R11[(int64_t)j * k + r] = Y[p * ldy + r];
    const int lpc = pick_lpc(L, MAXQ);
    const int cpw = 32 / lpc, sg = lane / lpc, sl = lane % lpc;
    Top2 loc;
    top2_init(loc);
    // (a one-iteration-ahead cp.async prefetch of the next column segment was measured: no gain
    // — the early steps already stream at ~5.9 TB/s of read+write — so loads stay direct)
    const int64_t cstride = (int64_t)kQrcpWarps * cpw;
    for (int64_t c0 = c_lo + (int64_t)warp * cpw; c0 < c_hi; c0 += cstride) {
      const int64_t c = c0 + sg;
      // a lane group works only on a live, unchosen, non-pivot column; the shuffles below are
      // executed by the whole warp regardless (dead groups carry zeros)
      bool live = c < c_hi;
      if (live && c == p) {
        if (sl == 0) w.nu[p] = -1.0;  // chosen
        live = false;
      }
      if (live && w.nu[c] < 0.0) live = false;  // chosen at an earlier step
      double2* yc = Y + c * ldy + j0;
      double2 y[MAXQ];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int rr = sl + lpc * q;
        y[q] = make_double2(0.0, 0.0);
        if (live && rr < L) y[q] = yc[rr];
      }
      for (int i = 0; i <= t; ++i) apply_reflector<MAXQ>(y, sv[i], s_tau[i][0], s_tau[i][1], sl, lpc, L);
      double nn = 0.0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int rr = sl + lpc * q;
        if (rr > t && rr < L) {
          nn = __fma_rn(y[q].x, y[q].x, nn);
          nn = __fma_rn(y[q].y, y[q].y, nn);
        }
      }
      if (block_end && live) {
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int rr = sl + lpc * q;
          if (rr < L) yc[rr] = y[q];
        }
      }
      const double nu = __dsqrt_rn(group_sum(nn, lpc));
      if (live && sl == 0) {
        w.nu[c] = nu;
        top2_push(loc, nu, c);
      }
    }
    block_top2_publish(loc, (j + 1) & 1);
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[4 * j + 2] = globaltimer();
    grid_barrier(w.bar, (unsigned)nb * (++phase));
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[4 * j + 3] = globaltimer();
  }
  if (b == 0 && threadIdx.x == 0) {
    out.info[0] = 0;
    out.info[1] = k;
  }
}

size_t qrcp_work_bytes(int64_t n, int max_blocks) {
  return (size_t)n * sizeof(double) + (size_t)2 * 3 * max_blocks * sizeof(double) + 256;
}

template <int MAXQ>
static cudaError_t launch_qrcp(double2* Y, int64_t ldy, int l, int64_t n, int k, double tol_rel,
                               const QrcpOut& out, const QrcpWork& w, int num_sms,
                               cudaStream_t st) {
  const size_t smem = sizeof(double2) * kQB * MAXQ * 32;
  cudaError_t e = cudaFuncSetAttribute(k_qrcp<MAXQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_qrcp<MAXQ>, kQrcpThreads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  int blocks = num_sms * (occ < 2 ? occ : 2);
  if (blocks > w.max_blocks) blocks = w.max_blocks;
  const int64_t min_cols = 8;  // keep >= 8 columns per CTA on small n
  if ((int64_t)blocks * min_cols > n) blocks = (int)((n + min_cols - 1) / min_cols);
  if (blocks < 1) blocks = 1;
  e = cudaMemsetAsync(w.bar, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  QrcpOut o = out;
  QrcpWork ww = w;
  void* args[] = {&Y, &ldy, &l, &n, &k, &tol_rel, &o, &ww};
  return cudaLaunchCooperativeKernel((void*)k_qrcp<MAXQ>, dim3(blocks), dim3(kQrcpThreads), args,
                                     smem, st);
}

cudaError_t qrcp(double2* Y, int64_t ldy, int64_t l, int64_t n, int64_t k, double tol_rel,
                 const QrcpOut& out, const QrcpWork& w, int num_sms, cudaStream_t st) {
  const int li = (int)l, ki = (int)k;
  const int qneed = (li + 31) / 32;
#define RID_Q(QV) \
  if (qneed <= QV) return launch_qrcp<QV>(Y, ldy, li, n, ki, tol_rel, out, w, num_sms, st);
  RID_Q(1) RID_Q(2) RID_Q(3) RID_Q(4) RID_Q(5) RID_Q(6) RID_Q(8) RID_Q(9) RID_Q(12) RID_Q(17)
  RID_Q(24) RID_Q(32)
#undef RID_Q
  return cudaErrorInvalidValue;  // l > 1024 unsupported
}

// ---------------------------------------------------------------------------------------------
// Inverse of the dense upper-triangular R11 (k x k, column-major): column c of R11^{-1} by
// right-looking back-substitution on e_c ("solving Lv = w for triangular L"); one CTA
// per column, the right-hand side in shared memory.
// ---------------------------------------------------------------------------------------------
__global__ void k_tri_inverse(const double2* __restrict__ R11, int k, double2* __restrict__ Rinv) {
  extern __shared__ double2 bvec[];  // k
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < k; i += blockDim.x) bvec[i] = make_double2(i == c ? 1.0 : 0.0, 0.0);
  __syncthreads();
  for (int s = c; s >= 0; --s) {
    const double d = R11[(int64_t)s * k + s].x;  // real diagonal (beta)
    const double2 xs = make_double2(__ddiv_rn(bvec[s].x, d), __ddiv_rn(bvec[s].y, d));
    const double2* col = R11 + (int64_t)s * k;  // R11[0:s, s]
    __syncthreads();
    for (int i = threadIdx.x; i < s; i += blockDim.x) {
      const double2 r = col[i];
      double2 bi = bvec[i];
      bi.x = __fma_rn(-r.x, xs.x, __fma_rn(r.y, xs.y, bi.x));
      bi.y = __fma_rn(-r.x, xs.y, __fma_rn(-r.y, xs.x, bi.y));
      bvec[i] = bi;
    }
    if (threadIdx.x == 0) bvec[s] = xs;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    Rinv[(int64_t)c * k + i] = (i <= c) ? bvec[i] : make_double2(0.0, 0.0);
}

cudaError_t tri_inverse(const double2* R11, int64_t k, double2* Rinv, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  const size_t sm = (size_t)k * sizeof(double2);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_tri_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm);
    if (e != cudaSuccess) return e;
  }
  k_tri_inverse<<<(unsigned)k, 256, sm, st>>>(R11, (int)k, Rinv);
  return cudaGetLastError();
}

}  // namespace rid
