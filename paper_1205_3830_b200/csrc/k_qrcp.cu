// k_qrcp.cu — column-pivoted Householder QR of the sketch Y (l x n), k steps, one persistent
// cooperative kernel with one grid barrier per step.
//
// Paper: "a highly approximate QR factorization on the matrix Y ... Y ≈ QR" with a column
// permutation "so that the first k columns are linearly independent and contain the k most
// weighted vectors" (§2, Eqs. 8–9); the authors note Householder "should result
// in similar stability with only half the runtime" of their CGS (§3.2).
// Readings: R8 greedy max residual 2-norm pivot, ties -> lowest column index;
// R13 rank failure when nu_p < 1e-13 * max_c ||Y[:, c]||. Residual norms (R11 / R11'):
//   * k_qrcp and k_qrcp_smem (the default for sketches under 64 MB: C1-C3) recompute every nu
//     exactly from the updated column each step (no downdating), like the oracle;
//   * k_qrcp_ring (the blocked default for larger sketches: C4, C5) DOWNDATES,
//     nu_c^2 <- nu_c^2 - |R(j, c)|^2, and recomputes nu_c exactly only when it has cancelled below
//     kRecompTol = 1e-4 of its last exact value (LAPACK zlaqps's safeguard, stricter). The
//     downdate's relative error is <= j u / 1e-4 (~6e-10 at j = 512), far below the top-2 pivot
//     gaps of the configs (>= 1.8e-6), so J is unchanged there; on inputs whose top-2 gap falls
//     below ~1e-9 (rid_diag.tie_margin_min) J may differ from the exact kernels and the oracle.
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
#include <cstdlib>

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "rid_device.cuh"
#include "rid_internal.h"
#include "rid_tma.cuh"

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

// Grid barrier: the CTA's writes are ordered before thread 0's arrival by bar.sync, the arrival is
// a gpu-scope release reduction, the wait a gpu-scope acquire load (no full fences; the polling
// is unslept: one thread per CTA on one L2 line)
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    while (ld_acquire(bar) < target) {
    }
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
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 0] = globaltimer();
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
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 1] = globaltimer();

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
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 2] = globaltimer();
    grid_barrier(w.bar, (unsigned)nb * (++phase));
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 3] = globaltimer();
  }
  if (b == 0 && threadIdx.x == 0) {
    out.info[0] = 0;
    out.info[1] = k;
  }
}

// =============================================================================================
// Small sketches (C1–C3: 16·l·n well under the SMs' shared memory): the exact-recompute QR with
// every CTA's columns resident in shared memory for all k steps. Per step the only global traffic
// is the per-CTA candidate triple and one column: before each grid barrier every CTA writes its
// local best column (rows j+1..l-1, double-buffered by step parity) to a slot, so after the
// barrier every CTA builds the reflector from the winner's slot — the global pivot is always some
// CTA's local best. The trailing update and the exact norms run from shared memory; the columns
// go back to Y after the last step.
// =============================================================================================
//
// CLUSTER = true (k_qrcp_cluster, sketches of at most a few MB: C1): the grid is ONE thread-block
// cluster of up to 16 CTAs and the exchange moves from global memory to distributed shared
// memory: every CTA publishes its candidate triple and its best column into its OWN shared
// memory (double-buffered by step parity), the grid barrier becomes the cluster barrier
// (barrier.cluster arrive.release / wait.acquire), and the pivot reduction and the winner's
// column are read from the peers' shared memory (mapa / ld.shared::cluster). The arithmetic is
// unchanged: the same bits as the grid-wide kernel (tested).
template <int MAXQ, bool CLUSTER = false>
__global__ void __launch_bounds__(kQrcpThreads, 1)
    k_qrcp_smem(double2* __restrict__ Y, int64_t ldy, int l, int64_t n, int k, double tol_rel,
                QrcpOut out, QrcpWork w, int per) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char qs_raw[];
  double2* sv = reinterpret_cast<double2*>(qs_raw);                   // MAXQ*32: v_j, rows j..
  double* snu = reinterpret_cast<double*>(sv + MAXQ * 32);            // per (even): norms, -1 chosen
  double2* sy = reinterpret_cast<double2*>(snu + ((per + 1) & ~1));   // per x l: the columns
  // CLUSTER: the exchange, in this CTA's shared memory: 2 x l slot, 2 x 3 candidate (parity)
  double2* sslot = sy + (size_t)per * l;
  double* scand = reinterpret_cast<double*>(sslot + (CLUSTER ? 2 * l : 0));
  __shared__ double s_tau[2];
  __shared__ Top2 sred[kQrcpWarps];
  __shared__ long long s_p;
  __shared__ int s_stop, s_best;

  // rows per lane in the column passes: up to QP (more columns per warp at once, shorter
  // butterflies) — the column lives in shared memory, so only registers bound it
  constexpr int QP = MAXQ < 12 ? 12 : MAXQ;
  const int nb = gridDim.x, b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c_lo = (int64_t)b * per;
  const int ncol = (int)((c_lo + per < n) ? per : (n > c_lo ? n - c_lo : 0));
  double nu0max = 0.0;
  unsigned phase = 0;

  // where CTA q's candidates / slot of a parity live (global, or q's shared memory)
  auto cand_of = [&](int parity, int q) -> const double* {
    if constexpr (CLUSTER)
      return cg::this_cluster().map_shared_rank(scand + 3 * parity, (unsigned)q);
    else
      return w.cand + ((size_t)parity * w.max_blocks + q) * 3;
  };
  auto slot_of = [&](int parity, int q) -> double2* {
    if constexpr (CLUSTER)
      return cg::this_cluster().map_shared_rank(sslot + (size_t)parity * l, (unsigned)q);
    else
      return w.xslot + ((size_t)parity * w.max_blocks + q) * l;
  };
  auto exchange_barrier = [&]() {
    if constexpr (CLUSTER)
      cg::this_cluster().sync();
    else
      grid_barrier(w.bar, (unsigned)nb * (++phase));
  };

  // publish the CTA's (best, second, index) and copy its best column's rows r0..l-1 to the slot
  auto publish = [&](Top2 loc, int parity, int r0) {
    top2_warp(loc);
    if (lane == 0) sred[warp] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
      Top2 tt = sred[0];
      for (int q = 1; q < kQrcpWarps; ++q) top2_merge(tt, sred[q]);
      double* c = const_cast<double*>(cand_of(parity, b));
      c[0] = tt.b1;
      c[1] = tt.b2;
      c[2] = (double)tt.i1;
      s_best = (tt.b1 >= 0.0) ? (int)(tt.i1 - c_lo) : -1;
    }
    __syncthreads();
    const int bl = s_best;
    if (bl >= 0) {
      double2* slot = slot_of(parity, b);
      for (int r = r0 + threadIdx.x; r < l; r += kQrcpThreads) slot[r] = sy[(int64_t)bl * l + r];
    }
  };

  // ---- phase 0: load the CTA's columns, exact norms -------------------------------------------
  for (int q = threadIdx.x; q < ncol * l; q += kQrcpThreads) {
    const int cl = q / l, r = q - cl * l;
    sy[q] = Y[(c_lo + cl) * ldy + r];
  }
  __syncthreads();
  {
    const int lpc = pick_lpc(l, QP);
    const int cpw = 32 / lpc, sg = lane / lpc, sl = lane % lpc;
    Top2 loc;
    top2_init(loc);
    for (int c0 = warp * cpw; c0 < ncol; c0 += kQrcpWarps * cpw) {
      const int cl = c0 + sg;
      const bool live = cl < ncol;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        const int r = sl + lpc * q;
        if (live && r < l) {
          const double2 y = sy[(int64_t)cl * l + r];
          s = __fma_rn(y.x, y.x, s);
          s = __fma_rn(y.y, y.y, s);
        }
      }
      const double nu = __dsqrt_rn(group_sum(s, lpc));
      if (live && sl == 0) {
        snu[cl] = nu;
        top2_push(loc, nu, c_lo + cl);
      }
    }
    publish(loc, 0, 0);
    exchange_barrier();
  }

  for (int j = 0; j < k; ++j) {
    const int L = l - j;  // rows j..l-1
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 0] = globaltimer();
    // ---- 1. global pivot (every CTA, identically) -----------------------------------------
    if (warp == 0) {
      Top2 tt;
      top2_init(tt);
      for (int q = lane; q < nb; q += 32) {
        const double* cb = cand_of(j & 1, q);
        Top2 o;
        o.b1 = cb[0];
        o.b2 = cb[1];
        o.i1 = (long long)cb[2];
        top2_merge(tt, o);
      }
      top2_warp(tt);
      if (j == 0) nu0max = tt.b1;
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
      // (CLUSTER: every CTA stops at the same step; no peer reads this CTA's shared memory after
      // the barrier it passed, and a CTA only exits after all peers' reads of its memory)
      if constexpr (CLUSTER) cg::this_cluster().sync();
      return;
    }
    const int64_t p = s_p;
    const int bp = (int)(p / per);  // the winner CTA: p was its local best

    // ---- 2. reflector H_j from the winner's slot (rows j..l-1 of column p) -------------------
    if (warp == 0) {
      const double2* xs = slot_of(j & 1, bp) + j;
      double2 x[MAXQ];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int rr = lane + 32 * q;
        x[q] = (rr < L) ? xs[rr] : make_double2(0.0, 0.0);
      }
      double s2 = 0.0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int rr = lane + 32 * q;
        if (rr > 0 && rr < L) {
          s2 = __fma_rn(x[q].x, x[q].x, s2);
          s2 = __fma_rn(x[q].y, x[q].y, s2);
        }
      }
      const double xnorm2 = group_sum(s2, 32);
      const double ar = __shfl_sync(0xffffffffu, x[0].x, 0), ai = __shfl_sync(0xffffffffu, x[0].y, 0);
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
          if (rr == 0) {
            v = make_double2(1.0, 0.0);
          } else {
            v.x = __fma_rn(x[q].x, sc_re, -__dmul_rn(x[q].y, sc_im));
            v.y = __fma_rn(x[q].x, sc_im, __dmul_rn(x[q].y, sc_re));
          }
          sv[rr] = v;
        }
      }
      if (lane == 0) {
        s_tau[0] = tau_re;
        s_tau[1] = tau_im;
        if (b == 0) {
          out.beta[j] = beta;
          out.R11[(int64_t)j * k + j] = make_double2(beta, 0.0);
        }
      }
    } else if (warp == 1 && b == bp) {
      // the owner: column p is chosen; rows 0..j-1 are final R entries
      const int pl = (int)(p - c_lo);
      if (lane == 0) snu[pl] = -1.0;
      for (int r = lane; r < j; r += 32) out.R11[(int64_t)j * k + r] = sy[(int64_t)pl * l + r];
    }
    __syncthreads();
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 1] = globaltimer();

    // ---- 3. every owned unchosen column in shared memory: apply H_j, exact norm --------------
    const double tr = s_tau[0], ti = s_tau[1];
    const int lpc = pick_lpc(L, QP);
    const int cpw = 32 / lpc, sg = lane / lpc, sl = lane % lpc;
    Top2 loc;
    top2_init(loc);
    for (int c0 = warp * cpw; c0 < ncol; c0 += kQrcpWarps * cpw) {
      const int cl = c0 + sg;
      const bool live = cl < ncol && snu[cl] >= 0.0;
      double2* yc = sy + (int64_t)(cl < ncol ? cl : 0) * l + j;
      double2 y[QP];
      double wr = 0.0, wi = 0.0;
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        const int rr = sl + lpc * q;
        y[q] = make_double2(0.0, 0.0);
        if (live && rr < L) {
          y[q] = yc[rr];
          const double2 vv = sv[rr];
          wr = __fma_rn(vv.x, y[q].x, __fma_rn(vv.y, y[q].y, wr));  // conj(v) y
          wi = __fma_rn(vv.x, y[q].y, __fma_rn(-vv.y, y[q].x, wi));
        }
      }
      wr = group_sum(wr, lpc);
      wi = group_sum(wi, lpc);
      const double s_re = __fma_rn(tr, wr, __dmul_rn(ti, wi));  // s = conj(tau) w
      const double s_im = __fma_rn(tr, wi, -__dmul_rn(ti, wr));
      double nn = 0.0;
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        const int rr = sl + lpc * q;
        if (live && rr < L) {
          const double2 vv = sv[rr];
          y[q].x = __fma_rn(-s_re, vv.x, __fma_rn(s_im, vv.y, y[q].x));  // y -= s v
          y[q].y = __fma_rn(-s_re, vv.y, __fma_rn(-s_im, vv.x, y[q].y));
          yc[rr] = y[q];
          if (rr > 0) {
            nn = __fma_rn(y[q].x, y[q].x, nn);
            nn = __fma_rn(y[q].y, y[q].y, nn);
          }
        }
      }
      const double nu = __dsqrt_rn(group_sum(nn, lpc));
      if (live && sl == 0) {
        snu[cl] = nu;
        top2_push(loc, nu, c_lo + cl);
      }
    }
    publish(loc, (j + 1) & 1, j + 1);
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 2] = globaltimer();
    exchange_barrier();
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 3] = globaltimer();
  }
  // ---- the columns go back: rows 0..k-1 hold R (R12 for the solve), the rest the residual ----
  for (int q = threadIdx.x; q < ncol * l; q += kQrcpThreads) {
    const int cl = q / l, r = q - cl * l;
    Y[(c_lo + cl) * ldy + r] = sy[q];
  }
  if (b == 0 && threadIdx.x == 0) {
    out.info[0] = 0;
    out.info[1] = k;
  }
  // CLUSTER: the last step's candidates are not read; no peer touches this CTA's memory now
}

// =============================================================================================
// Blocked variant (default): LAPACK zlaqps-style panels of nb <= kNB reflectors.
//
// The exact-recompute kernel above reads AND writes the whole trailing block every step (C4:
// ≈146 GB over 512 steps). Inside a panel starting at step j0 this kernel never rewrites the
// trailing block: with y^(j0)_c the column at the panel start and f_s(c) = conj(τ_s)·v_sᴴ y^(j0+s)_c,
//     y^(j+1)_c = y^(j0)_c − Σ_{s<=t} v_s f_s(c),         t = j − j0,
//     f_t(c)   = conj(τ_t)·( v_tᴴ y^(j0)_c − Σ_{s<t} (v_tᴴ v_s) f_s(c) ),
//     R(j, c)  = y^(j0)_c[j] − Σ_{s<=t} V[j, s] f_s(c),
// so step j reads rows j..l−1 of every trailing column once (the GEMV v_tᴴ y^(j0)), writes one
// element (R(j, c)) and one f per column, and downdates the residual norm
//     ν_c² ← ν_c² − |R(j, c)|²          (H_j is unitary on rows j..l−1)
// with the LAPACK safeguard: when (ν_new/ν_ref)² <= kRecompTol (ν_ref = the last exact value) the
// norm is recomputed exactly from y^(j0) (still in registers) minus the pending reflectors. The
// downdate's relative error is bounded by ≈ j·u/kRecompTol ≈ 6e-10 at j = 512 — four orders below
// the smallest top-2 pivot gap measured on C2–C5 (1.8e-6), so J is unaffected (R11').
// After each panel the trailing rows j0+nb..l−1 are updated in one tensor-core GEMM,
// Y −= V·F (k_zgemm.cu mode 2, K = nb): read + write once per nb steps instead of every step.
// =============================================================================================
constexpr int kNB = 16;         // max reflectors per panel (storage)
constexpr int kNBDefault = 16;  // panel width (measured on B200: nb = 24, 32 are slower at C4/C5)
constexpr double kRecompTol = 1e-4;
constexpr int kRingThreads = 256;
constexpr int kRingWarps = kRingThreads / 32;
constexpr int kMaxSlots = 64;
constexpr int kCH = 16;  // rows per streamed box (a box is kCH rows x 32 columns, 8 KB)

__device__ __forceinline__ void cmac_sub(double2& x, const double2 v, const double2 f) {  // x -= v f
  x.x = __fma_rn(-v.x, f.x, __fma_rn(v.y, f.y, x.x));
  x.y = __fma_rn(-v.x, f.y, __fma_rn(-v.y, f.x, x.y));
}
__device__ __forceinline__ void cmac_add(double& ar, double& ai, const double2 g, const double2 f) {
  ar = __fma_rn(g.x, f.x, __fma_rn(-g.y, f.y, ar));  // a += g f
  ai = __fma_rn(g.x, f.y, __fma_rn(g.y, f.x, ai));
}

__device__ __forceinline__ void consumers_sync() {  // warps 1..15 only
  asm volatile("bar.sync 1, %0;\n" ::"n"((kRingWarps - 1) * 32) : "memory");
}

// One CTA per SM, 8 warps (255 registers per thread). Warp 0: the pivot reduction. Warps 1..7:
// the reflector (every CTA builds the same one); then up to `ncw` of them each stream batches of
// 32 consecutive trailing columns as 16-row x 32-column boxes (2D TMA, 8 KB, completion on a
// slot's mbarrier, D boxes in flight per warp) and reduce them: inside a box lane = (row, column
// parity) with one register accumulator per column; at the end of a batch the partials are
// transposed through the consumed slot and lane i finishes column i (f_t, R(j, c), the downdated
// norm). Batches and rows are visited in alternating order from step to step (L2 reuse), and
// boxes past the first l2_keep bytes of the trailing block carry an evict_first policy.
//
// Sharding (NEXT-3): the grid is G rank groups of cpr CTAs; rank g's CTAs own rank g's columns
// (sh.Y[g], sh.w[g]) and nothing else of that rank is read by another rank except the pivot
// column of a step (from its owner's block, by every CTA, as the one-rank kernel reads it). The
// per-CTA candidates carry GLOBAL column ids, so the argmax (ties -> lowest global index) and
// every column's arithmetic are those of the one-rank kernel: any G gives the same bits.
struct RingMaps {
  CUtensorMap m[kQrMaxRanks];  // rank g's Y block as a (2l doubles) x n_loc matrix
};

template <int MAXQ>
__global__ void __launch_bounds__(kRingThreads, 1)
    k_qrcp_ring(const __grid_constant__ QrShards sh, int64_t ldy, int l, int k, int j0, int jend,
                double tol_rel, int ncw, int D, int per, int cpr, double l2_keep,
                const __grid_constant__ RingMaps tm) {
  constexpr int kCW = kRingWarps - 1;  // consumer warps in the reflector phase
  constexpr int kRQ = (MAXQ * 32 + kCW * 32 - 1) / (kCW * 32);
  extern __shared__ __align__(128) unsigned char ring_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ring_smem);                 // kMaxSlots
  double2* sv = reinterpret_cast<double2*>(full + kMaxSlots);              // MAXQ*32
  double2* ring = reinterpret_cast<double2*>(                              // ncw*D*32*kCH
      (reinterpret_cast<uintptr_t>(sv + MAXQ * 32 + 32) + 127) & ~(uintptr_t)127);  // TMA: 128 B
  __shared__ double2 s_vrow[kNB], s_g[kNB], s_fp[kNB];
  __shared__ double s_red[kRingWarps];
  __shared__ double s_par[2];  // alpha re/im
  __shared__ Top2 sred[kRingWarps];
  __shared__ long long s_p;
  __shared__ int s_stop;

  const int nbk = gridDim.x, b = blockIdx.x;
  const int g = b / cpr, bl = b - g * cpr;  // rank group and block within it
  double2* __restrict__ Y = sh.Y[g];
  const QrcpOut& out = sh.out[g];
  const QrcpWork& w = sh.w[g];
  const CUtensorMap& tmap = tm.m[g];
  double* const cand = sh.w[0].cand;  // the exchange: every CTA's candidates, all ranks
  unsigned* const bar = sh.w[0].bar;
  const int max_blocks = sh.w[0].max_blocks;
  const int64_t n = sh.n_loc;                    // this rank's columns (local ids 0..n-1)
  const int64_t gbase = (int64_t)g * sh.n_loc;   // global id of local column 0
  const int64_t nglob = (int64_t)sh.G * sh.n_loc;
  if (out.info[0] == 2) return;  // an earlier panel stopped on rank failure (uniform)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c_lo = (int64_t)bl * per;
  const int64_t c_hi = (c_lo + per < n) ? c_lo + per : n;
  const int64_t ldv = l;
  double nu0max = (j0 > 0) ? w.scal[0] : 0.0;
  unsigned phase = 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ncw * D; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (j0 == 0) {  // ---- initial exact column norms (one pass, direct loads) -------------------
    const int lpc = pick_lpc(l, MAXQ);
    const int cpw = 32 / lpc, sg = lane / lpc, sl = lane % lpc;
    Top2 loc;
    top2_init(loc);
    for (int64_t c0 = c_lo + (int64_t)warp * cpw; c0 < c_hi; c0 += (int64_t)kRingWarps * cpw) {
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
        w.nuref[c] = nu;
        top2_push(loc, nu, gbase + c);
      }
    }
    top2_warp(loc);
    if (lane == 0) sred[warp] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
      Top2 tt = sred[0];
      for (int q = 1; q < kRingWarps; ++q) top2_merge(tt, sred[q]);
      double* c = cand + (size_t)b * 3;  // parity 0
      c[0] = tt.b1;
      c[1] = tt.b2;
      c[2] = (double)tt.i1;
    }
    grid_barrier(bar, (unsigned)nbk * (++phase));
  }

  unsigned ubase = 0;  // items this warp streamed in earlier steps of this launch (ring parity)
  for (int j = j0; j < jend; ++j) {
    const int t = j - j0;
    const int L = l - j;  // rows j..l-1
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 0] = globaltimer();
    // ---- 1. global pivot (every CTA, identically); the owner marks it chosen --------------
    if (warp == 0) {
      Top2 tt;
      top2_init(tt);
      const double* cb = cand + (size_t)(j & 1) * max_blocks * 3;
      for (int q = lane; q < nbk; q += 32) {
        Top2 o;
        o.b1 = cb[q * 3 + 0];
        o.b2 = cb[q * 3 + 1];
        o.i1 = (long long)cb[q * 3 + 2];
        top2_merge(tt, o);
      }
      top2_warp(tt);
      if (j == 0) nu0max = tt.b1;  // max_c ||Y[:, c]||
      const bool stop =
          !(tt.b1 >= tol_rel * nu0max) || tt.b1 <= 0.0 || tt.i1 < 0 || tt.i1 >= nglob;
      const int64_t p = tt.i1;  // global id
      if (lane == 0) {
        s_p = p;
        s_stop = stop ? 1 : 0;
        if (bl == 0) {  // every rank's replicated outputs
          if (j == 0) w.scal[0] = nu0max;
          out.resid[j] = tt.b1;
          out.margin[j] = (tt.b2 < 0.0) ? DBL_MAX : (tt.b1 - tt.b2) / tt.b1;
          if (!stop) out.J[j] = p;
        }
      }
      if (!stop && p >= gbase + c_lo && p < gbase + c_hi && lane == 0)
        w.nu[p - gbase] = -1.0;  // the owner: chosen
    }
    __syncthreads();
    if (s_stop) {
      if (bl == 0 && threadIdx.x == 0) {
        out.info[0] = 2;
        out.info[1] = j;
      }
      return;  // no copy is in flight: every item of the previous step was consumed
    }
    // the pivot column lives in its owner's block: rows of y^(j0)_p and its f_s(p)
    const int64_t p = s_p;
    const int go = (int)(p / sh.n_loc);
    const int64_t pl = p - (int64_t)go * sh.n_loc;
    const double2* __restrict__ Yp = sh.Y[go] + pl * ldy;
    const double2* __restrict__ Fp = sh.w[go].F + pl * kNB;
    if (w.trace && b == 0 && threadIdx.x == 32) w.trace[8 * j + 4] = globaltimer();
    const bool rev = (j & 1) != 0;  // alternate the batch and row order (L2 reuse across steps)

    if (warp > 0) {
      const int cw = warp - 1, idx = cw * 32 + lane;
      // the CTA's columns are cut into batches of 32 consecutive columns (lane i <-> column i of
      // the batch; chosen columns leave their lane idle); streaming warp cw takes batches cw,
      // cw + ncw, ... and streams each batch's rows j..l-1 as kCH-row x 32-column boxes (one 2D
      // TMA copy of 8 KB per box, rows past l zero-filled) through its D ring slots
      const int nbat = (int)((c_hi - c_lo + 31) / 32);
      const int mybat = (cw < ncw && nbat > cw) ? (nbat - cw + ncw - 1) / ncw : 0;
      const int nch = (L + kCH - 1) / kCH;
      const int nitems = mybat * nch;
      // L2 residency: the first nkeep batches of every CTA (≈ l2_keep bytes of the trailing
      // block over the whole grid) are re-read from L2 at every step
      const double blk = 16.0 * (double)L * (double)nglob;  // all ranks' blocks share one L2
      const int nkeep = blk <= l2_keep ? nbat : (int)((double)nbat * l2_keep / blk);
      const uint64_t pol_first = policy_evict_first();
      // boxes are issued in consumption order, D ahead: (iq, ich) = batch and chunk of the next
      int iq = 0, ich = 0, isl = (int)(ubase % (unsigned)D), issued = 0;
      auto issue_next = [&]() {
        const int ch = rev ? nch - 1 - ich : ich;  // odd steps stream bottom-up
        const int bi = cw + ncw * iq;
        const int bb = rev ? nbat - 1 - bi : bi;
        const int s = cw * D + isl;
        if (lane == 0) {
          mbar_expect_tx(&full[s], (unsigned)(32 * kCH * sizeof(double2)));
          // batches below nkeep stay in L2 from step to step; the rest stream with evict_first
          if (bb < nkeep)
            tma_box_g2s(ring + (size_t)s * 32 * kCH, &tmap, 2 * (j + ch * kCH),
                        (int)(c_lo + 32 * bb), &full[s]);
          else
            tma_box_g2s_hint(ring + (size_t)s * 32 * kCH, &tmap, 2 * (j + ch * kCH),
                             (int)(c_lo + 32 * bb), &full[s], pol_first);
        }
        if (++ich == nch) {
          ich = 0;
          ++iq;
        }
        if (++isl == D) isl = 0;
      };
      // ---- 2a. prologue: this warp's first D boxes start streaming now ---------------------
      // (only the first box before the reflector: the rest would queue in front of its loads;
      // measured 0/1/2/3 boxes: C4 17.34/17.28/17.37/17.66 ms, C5 5.54/5.52/5.66/5.80 ms)
      for (; issued < nitems && issued < 1; ++issued) issue_next();
      // ---- 2b. reflector H_j from x = y^(j0)_p[j:l] − Σ_{s<t} V[j:l, s] f_s(p) --------------
      // all loads of a round are issued before their fmas: the pivot column's rows, then the
      // pending reflectors V[j:l, s] (8 columns per round) and f_s(p) (a broadcast)
      double2 x[kRQ];
      if constexpr (kRQ <= 3) {
#pragma unroll
      for (int q = 0; q < kRQ; ++q) {
        const int rr = idx + kCW * 32 * q;
        x[q] = rr < L ? Yp[j + rr] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int s0 = 0; s0 < kNB; s0 += 8) {
        if (s0 < t) {
          double2 vv[kRQ][8], fp[8];
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            fp[s] = s0 + s < t ? Fp[s0 + s] : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < kRQ; ++q) {
              const int rr = idx + kCW * 32 * q;
              vv[q][s] = (s0 + s < t && rr < L) ? w.V[(int64_t)(s0 + s) * ldv + j + rr]
                                                : make_double2(0.0, 0.0);
            }
          }
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            if (s0 + s < t) {
#pragma unroll
              for (int q = 0; q < kRQ; ++q) cmac_sub(x[q], vv[q][s], fp[s]);
              if (idx == 0) {  // row j: V[j, s] and f_s(p) for the column pass
                s_vrow[s0 + s] = vv[0][s];
                s_fp[s0 + s] = fp[s];
              }
            }
          }
        }
      }
      } else {  // l > 672: rows one at a time, 8 pending reflectors per round (registers)
#pragma unroll
        for (int q = 0; q < kRQ; ++q) {
          const int rr = idx + kCW * 32 * q;
          x[q] = rr < L ? Yp[j + rr] : make_double2(0.0, 0.0);
          for (int s0 = 0; s0 < t; s0 += 8) {
            double2 vv[8], fp[8];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              fp[s] = s0 + s < t ? Fp[s0 + s] : make_double2(0.0, 0.0);
              vv[s] = (s0 + s < t && rr < L) ? w.V[(int64_t)(s0 + s) * ldv + j + rr]
                                             : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              if (s0 + s < t) {
                cmac_sub(x[q], vv[s], fp[s]);
                if (idx == 0 && q == 0) {
                  s_vrow[s0 + s] = vv[s];
                  s_fp[s0 + s] = fp[s];
                }
              }
            }
          }
        }
      }
      double s2 = 0.0;
#pragma unroll
      for (int q = 0; q < kRQ; ++q) {
        const int rr = idx + kCW * 32 * q;
        if (rr > 0 && rr < L) {
          s2 = __fma_rn(x[q].x, x[q].x, s2);
          s2 = __fma_rn(x[q].y, x[q].y, s2);
        }
      }
      s2 = group_sum(s2, 32);
      if (lane == 0) s_red[cw] = s2;
      if (idx == 0) {
        s_par[0] = x[0].x;
        s_par[1] = x[0].y;
      }
      consumers_sync();
      if (w.trace && b == 0 && idx == 0) w.trace[8 * j + 5] = globaltimer();
      for (; issued < nitems && issued < D; ++issued) issue_next();  // the rest of the prologue
      double xnorm2 = 0.0;
      for (int q = 0; q < kCW; ++q) xnorm2 = __dadd_rn(xnorm2, s_red[q]);  // fixed order
      const double ar = s_par[0], ai = s_par[1];
      double tr, ti, beta, sc_re, sc_im;
      if (xnorm2 == 0.0 && ai == 0.0) {
        tr = 0.0;
        ti = 0.0;
        beta = ar;
        sc_re = 0.0;
        sc_im = 0.0;
      } else {
        const double nrm = __dsqrt_rn(__fma_rn(ar, ar, __fma_rn(ai, ai, xnorm2)));
        beta = (ar >= 0.0) ? -nrm : nrm;
        tr = __ddiv_rn(__dsub_rn(beta, ar), beta);
        ti = __ddiv_rn(-ai, beta);
        const double dr = __dsub_rn(ar, beta), di = ai;  // scal = 1 / (alpha - beta)
        const double den = __fma_rn(dr, dr, __dmul_rn(di, di));
        sc_re = __ddiv_rn(dr, den);
        sc_im = __ddiv_rn(-di, den);
      }
#pragma unroll
      for (int q = 0; q < kRQ; ++q) {
        const int rr = idx + kCW * 32 * q;
        if (rr < L) {
          double2 v;
          if (rr == 0) {
            v = make_double2(1.0, 0.0);
          } else {
            v.x = __fma_rn(x[q].x, sc_re, -__dmul_rn(x[q].y, sc_im));
            v.y = __fma_rn(x[q].x, sc_im, __dmul_rn(x[q].y, sc_re));
          }
          sv[rr] = v;
          if (bl == 0) w.V[(int64_t)t * ldv + j + rr] = v;  // each rank's copy of V
        }
      }
      if (idx < 32) sv[L + idx] = make_double2(0.0, 0.0);  // the last box reads up to L + 31
      if (bl == 0) {
        if (idx == 0) {
          out.beta[j] = beta;
          out.R11[(int64_t)j * k + j] = make_double2(beta, 0.0);
        }
      }
      consumers_sync();
      if (w.trace && b == 0 && idx == 0) w.trace[8 * j + 6] = globaltimer();
      // s_g[s] = v_tᴴ v_s for s < t (one warp per s)
      for (int s = cw; s < t; s += kCW) {
        const double2* vs = w.V + (int64_t)s * ldv + j;
        double gr = 0.0, gi = 0.0;
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int rr = lane + 32 * q;
          if (rr < L) {
            const double2 a = sv[rr], v = vs[rr];
            gr = __fma_rn(a.x, v.x, __fma_rn(a.y, v.y, gr));  // conj(a) v
            gi = __fma_rn(a.x, v.y, __fma_rn(-a.y, v.x, gi));
          }
        }
        gr = group_sum(gr, 32);
        gi = group_sum(gi, 32);
        if (lane == 0) s_g[s] = make_double2(gr, gi);
      }
      consumers_sync();
      if (w.trace && b == 0 && idx == 0) w.trace[8 * j + 1] = globaltimer();

      // ---- 3. this warp's batches. Inside a box lane = (row rl, column parity half): each lane
      // accumulates conj(v[row])·y over its row of 16 of the batch's columns (a register per
      // column, v in a register, one conflict-free 512 B shared-memory wavefront group per
      // column pair); at the end of a batch the partials are transposed through the consumed
      // slot and lane i sums column i's 16 row-partials in a fixed order. ------------------------
      const int rl = lane & (kCH - 1), half = lane >> 4;
      Top2 loc;
      top2_init(loc);
      bool live = false;
      int64_t c = 0;
      double nu_old = 0.0, ref = 0.0, hr = 0.0, hi = 0.0, rsr = 0.0, rsi = 0.0;
      double2 yj = make_double2(0.0, 0.0);
      double2 acc[16];
      int cq = 0, cch = 0, csl = (int)(ubase % (unsigned)D);
      unsigned cph = (ubase / (unsigned)D) & 1u;
      for (int u = 0; u < nitems; ++u) {
        const int ch = rev ? nch - 1 - cch : cch;
        if (cch == 0) {  // batch start: lane i's column, its norms, row j, pending-reflector terms
          const int bi = cw + ncw * cq;
          const int bb = rev ? nbat - 1 - bi : bi;
          c = c_lo + 32 * bb + lane;
          nu_old = c < c_hi ? w.nu[c] : -1.0;
          live = nu_old >= 0.0;  // chosen columns (and p) carry -1
          ref = live ? w.nuref[c] : 0.0;
          yj = live ? Y[c * ldy + j] : make_double2(0.0, 0.0);
          // h = Σ_{s<t} g_s f_s,  rs = Σ_{s<t} V[j, s] f_s
          hr = hi = rsr = rsi = 0.0;
#pragma unroll
          for (int s0 = 0; s0 < kNB; s0 += 8) {
            double2 f[8];
#pragma unroll
            for (int s = 0; s < 8; ++s)
              f[s] = (live && s0 + s < t) ? w.F[c * kNB + s0 + s] : make_double2(0.0, 0.0);
#pragma unroll
            for (int s = 0; s < 8; ++s)
              if (s0 + s < t) {
                cmac_add(hr, hi, s_g[s0 + s], f[s]);
                cmac_add(rsr, rsi, s_vrow[s0 + s], f[s]);
              }
          }
#pragma unroll
          for (int cc = 0; cc < 16; ++cc) acc[cc] = make_double2(0.0, 0.0);
        }
        const int s = cw * D + csl;
        mbar_wait(&full[s], cph);
        double2* box = ring + (size_t)s * 32 * kCH;  // [32 columns][kCH rows]
        const double2 v = sv[ch * kCH + rl];
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) {
          const double2 y = box[(2 * cc + half) * kCH + rl];
          acc[cc].x = __fma_rn(v.x, y.x, __fma_rn(v.y, y.y, acc[cc].x));  // conj(v) y
          acc[cc].y = __fma_rn(v.x, y.y, __fma_rn(-v.y, y.x, acc[cc].y));
        }
        const bool last = cch == nch - 1;
        double dr = 0.0, di = 0.0;
        __syncwarp();
        if (last) {  // transpose through the consumed slot: lane i sums column i
#pragma unroll
          for (int cc = 0; cc < 16; ++cc) box[(2 * cc + half) * kCH + rl] = acc[cc];
          __syncwarp();
          double e0r = 0.0, e0i = 0.0, e1r = 0.0, e1i = 0.0;
#pragma unroll
          for (int r = 0; r < kCH; r += 2) {
            const double2 p0 = box[lane * kCH + ((r + lane) & (kCH - 1))];
            const double2 p1 = box[lane * kCH + ((r + 1 + lane) & (kCH - 1))];
            e0r = __dadd_rn(e0r, p0.x);
            e0i = __dadd_rn(e0i, p0.y);
            e1r = __dadd_rn(e1r, p1.x);
            e1i = __dadd_rn(e1i, p1.y);
          }
          dr = __dadd_rn(e0r, e1r);
          di = __dadd_rn(e0i, e1i);
          __syncwarp();
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic -> TMA (WAR)
        __syncwarp();
        if (issued < nitems) {  // refill the slot D boxes ahead
          issue_next();
          ++issued;
        }
        if (last && live) {  // ---- lane i's column is complete --------------------------------
          dr = __dsub_rn(dr, hr);  // d = v_tᴴ y − h
          di = __dsub_rn(di, hi);
          const double2 ft = make_double2(__fma_rn(tr, dr, __dmul_rn(ti, di)),  // conj(tau) d
                                          __fma_rn(tr, di, -__dmul_rn(ti, dr)));
          const double2 Rj = make_double2(__dsub_rn(__dsub_rn(yj.x, rsr), ft.x),
                                          __dsub_rn(__dsub_rn(yj.y, rsi), ft.y));
          // downdate ν² ← ν² − |R(j, c)|²; exact recompute when it has cancelled below
          // kRecompTol·ν_ref² (LAPACK zlaqps safeguard)
          const double d2 =
              __fma_rn(-Rj.x, Rj.x, __fma_rn(-Rj.y, Rj.y, __dmul_rn(nu_old, nu_old)));
          const bool need = !(nu_old > 0.0) || !(d2 > kRecompTol * __dmul_rn(ref, ref));
          double nu_new = __dsqrt_rn(d2 > 0.0 ? d2 : 0.0);
          if (need) {  // rare, this lane alone: rows j+1..l-1 of y^(j+1) from global memory
            double nn = 0.0;
            for (int rr = 1; rr < L; ++rr) {
              double2 z = Y[c * ldy + j + rr];
              for (int uu = 0; uu < t; ++uu)
                cmac_sub(z, w.V[(int64_t)uu * ldv + j + rr], w.F[c * kNB + uu]);
              cmac_sub(z, sv[rr], ft);
              nn = __fma_rn(z.x, z.x, nn);
              nn = __fma_rn(z.y, z.y, nn);
            }
            nu_new = __dsqrt_rn(nn);
          }
          w.F[c * kNB + t] = ft;
          Y[c * ldy + j] = Rj;
          w.nu[c] = nu_new;
          if (need) w.nuref[c] = nu_new;
          top2_push(loc, nu_new, gbase + c);
        }
        if (++cch == nch) {
          cch = 0;
          ++cq;
        }
        if (++csl == D) {
          csl = 0;
          cph ^= 1u;
        }
      }
      ubase += (unsigned)nitems;
      top2_warp(loc);
      if (lane == 0) sred[warp] = loc;
    } else {
      // warp 0 is idle while warps 1.. build the reflector and stream: CTA 0's copies rows
      // 0..j-1 of the pivot column (final R entries) into the dense R11 off the critical path
      if (bl == 0)  // every rank's copy, from the owner's block
        for (int r = lane; r < j; r += 32) out.R11[(int64_t)j * k + r] = Yp[r];
      if (lane == 0) {
        Top2 z;
        top2_init(z);
        sred[0] = z;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Top2 tt = sred[0];
      for (int q = 1; q < kRingWarps; ++q) top2_merge(tt, sred[q]);
      double* cc = cand + ((size_t)((j + 1) & 1) * max_blocks + b) * 3;
      cc[0] = tt.b1;
      cc[1] = tt.b2;
      cc[2] = (double)tt.i1;
    }
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 2] = globaltimer();
    if (j + 1 < jend) grid_barrier(bar, (unsigned)nbk * (++phase));
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 3] = globaltimer();
  }
  if (bl == 0 && threadIdx.x == 0) out.info[1] = jend;
}

// =============================================================================================
// Lazy-refresh blocked variant (default for blocked sketches with 384 < l <= 544: C4).
//
// The ring kernel above streams rows j..l−1 of EVERY unchosen column at every step (C4: 73 GB
// over 512 steps) because the greedy rule (R8) needs the exact maximum residual norm. But a
// residual norm never grows (ν_c(j+1)² = ν_c(j)² − |R(j, c)|²): a norm computed at an earlier
// step of the panel is an UPPER BOUND on the current one, and a column whose bound is below the
// current maximum cannot be the pivot. This kernel keeps, per column, the number u of panel steps
// already applied to it (f_0..f_{u−1}(c) in F, R(j0..j0+u−1, c) in Y, ν_c exact as of step j0+u)
// and at step j refreshes ONLY the columns whose bound is >= a threshold τ_j:
//   phase A (FP64 tensor pipe, 8 columns x 16 reflectors per DMMA tile): d_s = v_sᴴ y^(j0)_c for
//     s = u..t, V of the panel in shared memory, y^(j0)_c[j0+u:l] read once from global memory;
//   phase B (a half-warp per column): for s = u..t in order
//       f_s = conj(τ_s)·(d_s − Σ_{s'<s} (v_sᴴ v_s') f_s')   (as f = M d, M built once per step),
//       R(j0+s, c) = y^(j0)_c[j0+s] − Σ_{s'<=s} V[j0+s, s'] f_s',
//       ν² ← ν² − |R(j0+s, c)|²  (exact recompute below kRecompTol·ν_ref², as the ring kernel).
// A column's arithmetic is fixed (fixed lanes, fixed reduction orders, the same per-s formulas),
// so WHEN it is refreshed changes no bit: J, R, P and the norms equal those of refreshing every
// column at every step (mode 2, RID_QRCP_LAZY=2; tested bitwise).
// Exact pivots: the exchange after a pass carries the grid-wide top three of the refreshed
// columns' exact norms (b1, b2, b3) and m, the largest bound of the columns NOT refreshed at this
// step; their exact norms are <= m. If b2 > m the top two are exact (the argmax, ties to the
// lowest index, and the tie margin); otherwise the pass is repeated down to b2 (or to m with fewer
// than two exact norms), which terminates. The threshold on ν², τ_j = b3(j)·(1 − κ/(l − j)):
// the third-best norm less κ mean one-step decays of a residual in l − j dimensions (κ = 8), so
// the next top two are usually among the refreshed columns. The last step of a
// launch refreshes every column (τ = −1): the trailing update Y −= V·F needs all of f_0..f_{nb−1}
// and rows j0..jend−1 of every column must hold R.
// =============================================================================================
constexpr int kLazyThreads = 256;
constexpr int kLazyWarps = kLazyThreads / 32;
constexpr int kLazyChunk = 128;  // columns per phase A / phase B round (s_d rows)
constexpr int kLazySD = kNB + 1;  // s_d row stride in double2 (conflict-free 16-byte rows)
constexpr int kLazyScratch = 8 * 2 * 4 * 32 * 2;  // phase A partials [pp][mt][prod][lane][2]

// Top three exact norms (ties of the first to the lowest index) and the largest bound among the
// columns NOT refreshed at this step (m): the exchange record of the lazy kernel.
struct Top3 {
  double b1, b2, b3, m;
  long long i1;
};
__device__ __forceinline__ void top3_init(Top3& a) {
  a.b1 = a.b2 = a.b3 = a.m = -1.0;
  a.i1 = 0x7FFFFFFFFFFFFFFFLL;
}
__device__ __forceinline__ void top3_push(Top3& a, double v, long long i) {
  if (beats(v, i, a.b1, a.i1)) {
    a.b3 = a.b2;
    a.b2 = a.b1;
    a.b1 = v;
    a.i1 = i;
  } else if (v > a.b2) {
    a.b3 = a.b2;
    a.b2 = v;
  } else if (v > a.b3) {
    a.b3 = v;
  }
}
// top three of the union (as multisets of values; the first by (value, -index)): order-free
__device__ __forceinline__ void top3_merge(Top3& a, const Top3& c) {
  const bool cw = beats(c.b1, c.i1, a.b1, a.i1);
  const Top3& w = cw ? c : a;  // holds the winner
  const Top3& o = cw ? a : c;
  Top3 r;
  r.b1 = w.b1;
  r.i1 = w.i1;
  if (o.b1 >= w.b2) {
    r.b2 = o.b1;
    r.b3 = fmax(w.b2, o.b2);
  } else {
    r.b2 = w.b2;
    r.b3 = fmax(w.b3, o.b1);
  }
  r.m = fmax(a.m, c.m);
  a = r;
}
__device__ __forceinline__ void top3_warp(Top3& a) {
#pragma unroll
  for (int msk = 16; msk >= 1; msk >>= 1) {
    Top3 o;
    o.b1 = __shfl_xor_sync(0xffffffffu, a.b1, msk);
    o.b2 = __shfl_xor_sync(0xffffffffu, a.b2, msk);
    o.b3 = __shfl_xor_sync(0xffffffffu, a.b3, msk);
    o.m = __shfl_xor_sync(0xffffffffu, a.m, msk);
    o.i1 = __shfl_xor_sync(0xffffffffu, a.i1, msk);
    top3_merge(a, o);
  }
}

template <int MAXQ>
__global__ void __launch_bounds__(kLazyThreads, 1)
    k_qrcp_lazy(const __grid_constant__ QrShards sh, int64_t ldy, int l, int k, int j0, int jend,
                double tol_rel, int per, int cpr, double kappa, int mode) {
  constexpr int RP = 32 * MAXQ + 4;  // sV row stride: rows j0..j0+32·MAXQ−1, +64 B so that the
                                      // DMMA A fragments (8 s x 4 rows) hit 32 distinct banks
  constexpr int XQ = (32 * MAXQ + kLazyThreads - 1) / kLazyThreads;
  constexpr int KQ = MAXQ;  // k-steps (4 rows) per partial: 8 partials x KQ x 4 >= 32 MAXQ
  extern __shared__ __align__(16) unsigned char lz_smem[];
  double2* sV = reinterpret_cast<double2*>(lz_smem);           // [kNB][RP]: v_s, zero above j0+s
  double2* s_d = sV + kNB * RP;                                 // [kLazyChunk][kLazySD]: d_s
  double* s_sc = reinterpret_cast<double*>(s_d + kLazyChunk * kLazySD);  // [8][8][64]
  double* nu_s = s_sc + kLazyScratch;                           // [per] ν² bound (exact at j0+u)
  double* ref_s = nu_s + per;                                   // [per] ν² at the last recompute
  int* upd_s = reinterpret_cast<int*>(ref_s + per);             // [per] u: panel steps applied
  int* list = upd_s + per;                                      // [per] the pass's columns
  __shared__ double2 s_G[kNB][kNB];  // s_G[t][s] = v_tᴴ v_s, s < t
  __shared__ double2 s_M[kNB][kNB + 1];  // f = M d: M = (I + D_conj(τ) G)^-1 D_conj(τ), lower
                                         // (padded: phase B's lanes read a column of it)
  __shared__ double2 s_fp[kNB];      // f_s(p) of the step's pivot
  __shared__ double s_red[kLazyWarps];
  __shared__ double s_par[2];
  __shared__ Top3 sred[kLazyWarps];
  __shared__ Top3 s_top;
  __shared__ int s_cnt;

  const int nbk = gridDim.x, b = blockIdx.x;
  const int g = b / cpr, bl = b - g * cpr;
  double2* __restrict__ Y = sh.Y[g];
  const QrcpOut& out = sh.out[g];
  const QrcpWork& w = sh.w[g];
  double* const cand = sh.w[0].cand;  // 2 buffers x max_blocks x 8 doubles
  unsigned* const bar = sh.w[0].bar;
  const int max_blocks = sh.w[0].max_blocks;
  const int64_t n = sh.n_loc;
  const int64_t gbase = (int64_t)g * sh.n_loc;
  const int64_t nglob = (int64_t)sh.G * sh.n_loc;
  if (out.info[0] == 2) return;  // an earlier panel stopped on rank failure (uniform)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c_lo = (int64_t)bl * per;
  const int ncol = (int)(n - c_lo < per ? (n - c_lo > 0 ? n - c_lo : 0) : per);
  const int64_t ldv = l;
  const int Lp = l - j0;          // rows of the panel
  const int qn = (Lp + 31) / 32;  // q < qn hold them
  const int nks = (Lp + 3) >> 2;  // 4-row k-steps of the panel
  unsigned phase = 0;
  int xc = (j0 > 0) ? (int)__ldcg(sh.w[0].scal + 1) : 0;  // cand buffer of the last exchange
  double nu0max = (j0 > 0) ? __ldcg(w.scal) : 0.0;

  for (int i = threadIdx.x; i < kNB * RP; i += kLazyThreads) sV[i] = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < ncol; i += kLazyThreads) {
    upd_s[i] = 0;
    if (j0 > 0) {
      nu_s[i] = __ldcg(w.nu + c_lo + i);
      ref_s[i] = __ldcg(w.nuref + c_lo + i);
    }
  }
  __syncthreads();

  int jx = -1;  // (trace) the step whose exchange is timed
  // grid-wide record of the last exchange -> s_top: every warp merges a slice of the records
  // (one per lane, two 16-byte loads), then thread 0 the eight warp results (order-free merges)
  auto read_top = [&]() {
    Top3 tt;
    top3_init(tt);
    const double* cb = cand + (size_t)xc * max_blocks * 8;
    for (int q = threadIdx.x; q < nbk; q += kLazyThreads) {
      const double2 v0 = __ldcg(reinterpret_cast<const double2*>(cb + q * 8));
      const double2 v1 = __ldcg(reinterpret_cast<const double2*>(cb + q * 8 + 2));
      Top3 o;
      o.b1 = v0.x;
      o.b2 = v0.y;
      o.b3 = v1.x;
      o.m = v1.y;
      o.i1 = (long long)__ldcg(cb + q * 8 + 4);
      top3_merge(tt, o);
    }
    top3_warp(tt);
    if (lane == 0) sred[warp] = tt;
    __syncthreads();
    if (threadIdx.x == 0) {
      Top3 a = sred[0];
      for (int q = 1; q < kLazyWarps; ++q) top3_merge(a, sred[q]);
      s_top = a;
    }
    __syncthreads();
  };
  // the CTA's record over its columns (exact: refreshed as of panel step tf), published; grid
  // barrier; the grid-wide record
  auto exchange = [&](int tf) {
    Top3 loc;
    top3_init(loc);
    for (int i = threadIdx.x; i < ncol; i += kLazyThreads) {
      const double v = nu_s[i];
      if (v >= 0.0) {
        if (upd_s[i] == tf)
          top3_push(loc, v, gbase + c_lo + i);
        else
          loc.m = fmax(loc.m, v);
      }
    }
    top3_warp(loc);
    if (lane == 0) sred[warp] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
      Top3 tt = sred[0];
      for (int q = 1; q < kLazyWarps; ++q) top3_merge(tt, sred[q]);
      double* cc = cand + ((size_t)(xc ^ 1) * max_blocks + b) * 8;  // 64-byte records
      reinterpret_cast<double2*>(cc)[0] = make_double2(tt.b1, tt.b2);
      reinterpret_cast<double2*>(cc)[1] = make_double2(tt.b3, tt.m);
      cc[4] = (double)tt.i1;
    }
    xc ^= 1;
    const unsigned long long tX0 = (w.trace && b == 0) ? globaltimer() : 0ull;
    grid_barrier(bar, (unsigned)nbk * (++phase));
    const unsigned long long tX1 = (w.trace && b == 0) ? globaltimer() : 0ull;
    read_top();
    if (w.trace && b == 0 && threadIdx.x == 0 && jx >= 0) {
      w.trace[8 * jx + 4] += tX1 - tX0;
      w.trace[8 * jx + 5] += globaltimer() - tX1;
    }
  };

  if (j0 == 0) {  // ---- initial exact column norms² (one warp per column) ----------------------
    for (int i = warp; i < ncol; i += kLazyWarps) {
      const double2* yc = Y + (c_lo + i) * ldy;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int r = lane + 32 * q;
        if (r < l) {
          const double2 y = __ldcg(yc + r);
          s = __fma_rn(y.x, y.x, s);
          s = __fma_rn(y.y, y.y, s);
        }
      }
      s = group_sum(s, 32);
      if (lane == 0) {
        nu_s[i] = s;
        ref_s[i] = s;
      }
    }
    __syncthreads();
    exchange(0);
  } else {
    read_top();
  }

  for (int j = j0; j < jend; ++j) {
    const int t = j - j0;
    const int L = l - j;
    jx = j;
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 0] = globaltimer();
    // ---- 1. the pivot (every CTA identically, from s_top; values are ν²) ---------------------
    const Top3 tt = s_top;
    const double nu1 = __dsqrt_rn(tt.b1 > 0.0 ? tt.b1 : 0.0);
    if (j == 0) nu0max = nu1;  // max_c ||Y[:, c]||
    const bool stop = !(nu1 >= tol_rel * nu0max) || tt.b1 <= 0.0 || tt.i1 < 0 || tt.i1 >= nglob;
    const int64_t p = tt.i1;  // global id
    if (bl == 0 && threadIdx.x == 0) {  // every rank's replicated outputs
      if (j == 0) w.scal[0] = nu0max;
      out.resid[j] = nu1;
      out.margin[j] = (tt.b2 < 0.0) ? DBL_MAX : (nu1 - __dsqrt_rn(tt.b2)) / nu1;
      if (!stop) out.J[j] = p;
    }
    if (stop) {
      if (bl == 0 && threadIdx.x == 0) {
        out.info[0] = 2;
        out.info[1] = j;
      }
      return;
    }
    // this step's refresh threshold on ν²: the third-best exact value less kappa mean one-step
    // decays of a residual in l − j dimensions (-1: every column)
    double tau = -1.0;
    if (mode != 2 && j + 1 < jend) {
      const double base = tt.b3 > 0.0 ? tt.b3 : tt.b2;
      const double dec = 1.0 - kappa / (double)(L > 1 ? L : 1);
      tau = (base > 0.0 && dec > 0.0) ? base * dec : -1.0;
    }
    const int go = (int)(p / sh.n_loc);
    const int64_t pl = p - (int64_t)go * sh.n_loc;
    const double2* __restrict__ Yp = sh.Y[go] + pl * ldy;
    if (threadIdx.x == 0 && p >= gbase + c_lo && p < gbase + c_lo + ncol)
      nu_s[p - gbase - c_lo] = -1.0;  // the owner: chosen
    if (threadIdx.x < t) s_fp[threadIdx.x] = __ldcg(sh.w[go].F + pl * kNB + threadIdx.x);
    __syncthreads();
    // ---- 2. reflector H_j from x = y^(j0)_p[j:l] − Σ_{s<t} V[j:l, s] f_s(p) ----------------
    double2 x[XQ];
    double s2 = 0.0;
#pragma unroll
    for (int q = 0; q < XQ; ++q) {
      const int rr = threadIdx.x + kLazyThreads * q;
      double2 z = make_double2(0.0, 0.0);
      if (rr < L) {
        z = __ldcg(Yp + j + rr);
        for (int s = 0; s < t; ++s) cmac_sub(z, sV[s * RP + t + rr], s_fp[s]);
        if (rr > 0) {
          s2 = __fma_rn(z.x, z.x, s2);
          s2 = __fma_rn(z.y, z.y, s2);
        }
      }
      x[q] = z;
    }
    s2 = group_sum(s2, 32);
    if (lane == 0) s_red[warp] = s2;
    if (threadIdx.x == 0) {
      s_par[0] = x[0].x;
      s_par[1] = x[0].y;
    }
    if (bl == 0)  // R11 column j: rows 0..j-1 of the pivot are final
      for (int r = threadIdx.x; r < j; r += kLazyThreads) out.R11[(int64_t)j * k + r] = __ldcg(Yp + r);
    __syncthreads();
    {
      double xnorm2 = 0.0;
      for (int q = 0; q < kLazyWarps; ++q) xnorm2 = __dadd_rn(xnorm2, s_red[q]);  // fixed order
      const double ar = s_par[0], ai = s_par[1];
      double tr, ti, beta, sc_re, sc_im;
      if (xnorm2 == 0.0 && ai == 0.0) {
        tr = 0.0;
        ti = 0.0;
        beta = ar;
        sc_re = 0.0;
        sc_im = 0.0;
      } else {
        const double nrm = __dsqrt_rn(__fma_rn(ar, ar, __fma_rn(ai, ai, xnorm2)));
        beta = (ar >= 0.0) ? -nrm : nrm;
        tr = __ddiv_rn(__dsub_rn(beta, ar), beta);
        ti = __ddiv_rn(-ai, beta);
        const double dr = __dsub_rn(ar, beta), di = ai;  // scal = 1 / (alpha - beta)
        const double den = __fma_rn(dr, dr, __dmul_rn(di, di));
        sc_re = __ddiv_rn(dr, den);
        sc_im = __ddiv_rn(-di, den);
      }
#pragma unroll
      for (int q = 0; q < XQ; ++q) {
        const int rr = threadIdx.x + kLazyThreads * q;
        if (rr < L) {
          double2 v;
          if (rr == 0) {
            v = make_double2(1.0, 0.0);
          } else {
            v.x = __fma_rn(x[q].x, sc_re, -__dmul_rn(x[q].y, sc_im));
            v.y = __fma_rn(x[q].x, sc_im, __dmul_rn(x[q].y, sc_re));
          }
          sV[t * RP + t + rr] = v;
          if (bl == 0) w.V[(int64_t)t * ldv + j + rr] = v;  // each rank's copy (trailing update)
        }
      }
      if (threadIdx.x == 0) {
        s_M[t][t] = make_double2(tr, -ti);  // conj(τ_t)
        if (bl == 0) {
          out.beta[j] = beta;
          out.R11[(int64_t)j * k + j] = make_double2(beta, 0.0);
        }
      }
    }
    __syncthreads();
    // s_G[t][s] = v_tᴴ v_s for s < t (one warp per s, rows on fixed lanes)
    for (int s = warp; s < t; s += kLazyWarps) {
      double gr = 0.0, gi = 0.0;
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        if (q < qn) {
          const double2 a = sV[t * RP + lane + 32 * q], v = sV[s * RP + lane + 32 * q];
          gr = __fma_rn(a.x, v.x, __fma_rn(a.y, v.y, gr));  // conj(a) v
          gi = __fma_rn(a.x, v.y, __fma_rn(-a.y, v.x, gi));
        }
      }
      gr = group_sum(gr, 32);
      gi = group_sum(gi, 32);
      if (lane == 0) s_G[t][s] = make_double2(gr, gi);
    }
    __syncthreads();
    // row t of M: f_t = conj(τ_t)(d_t − Σ_{s<t} G[t][s] f_s) with f_s = Σ_{s'<=s} M[s][s'] d_s',
    // so M[t][s'] = −conj(τ_t) Σ_{s'<=s<t} G[t][s] M[s][s'] (one thread per s', fixed order)
    if (threadIdx.x < t) {
      const int sp = threadIdx.x;
      double ar = 0.0, ai = 0.0;
      for (int s = sp; s < t; ++s) cmac_add(ar, ai, s_G[t][s], s_M[s][sp]);
      const double2 ct = s_M[t][t];
      s_M[t][sp] = make_double2(-__fma_rn(ct.x, ar, -__dmul_rn(ct.y, ai)),
                                -__fma_rn(ct.x, ai, __dmul_rn(ct.y, ar)));
    }
    __syncthreads();
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 1] = globaltimer();

    // ---- 3. the pass: refresh every live column whose bound is >= thr ------------------------
    auto pass = [&](double thr) {
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < ncol; i += kLazyThreads) {
        const double v = nu_s[i];
        if (v >= 0.0 && upd_s[i] <= t && v >= thr) list[atomicAdd(&s_cnt, 1)] = i;
      }
      __syncthreads();
      const int cnt = s_cnt;
      if (w.trace && threadIdx.x == 0 && cnt > 0)
        atomicAdd(&w.trace[8 * j + 6], (unsigned long long)cnt);
      for (int e0 = 0; e0 < cnt; e0 += kLazyChunk) {
        const int nch = min(kLazyChunk, cnt - e0);
        // phase A on the FP64 tensor pipe: d_s(c) = v_sᴴ y^(j0)_c for 8 columns x 16 s per tile
        // (DMMA m8n8k4: A = V from shared memory, B = Y straight from global memory), K = the
        // panel rows in 4-row steps; step κ goes to partial κ mod 8 (the eight warps of a tile:
        // short chains for the few-column lazy passes), and each of the four real products
        // Vx·Yx, Vy·Yy, Vx·Yy, Vy·Yx is its own ascending DMMA chain (eight independent chains per
        // warp: the DMMA latency is ≈ 8 issues deep); per product the eight partials summed
        // pairwise in a fixed tree, then Re d = XX + YY, Im d = XY − YX. Per (s, c) the bits
        // depend only on v_s and y_c: not on the tile, the pass or the other columns. The next
        // tile's loads are issued before the combine.
        const int ntile = (nch + 7) / 8;
        const int pp = warp, gq = lane >> 2, tq = lane & 3;  // warp = partial
        double2 yv[KQ];
        int uc = kNB;
        auto load_tile = [&](int tl) {
          const int ecol = tl * 8 + gq;  // this lane's B column (chunk entry)
          const bool cv = tl < ntile && ecol < nch;
          const int ic = cv ? list[e0 + ecol] : 0;
          uc = cv ? upd_s[ic] : kNB;
          const double2* yc = Y + (c_lo + ic) * ldy + j0;
#pragma unroll
          for (int i = 0; i < KQ; ++i) {
            const int r = 4 * (pp + 8 * i) + tq;
            // rows >= u of y^(j0) are not written during this launch (only rows j0..j0+u−1
            // receive R), so the read-only path is coherent for every row read here
            yv[i] = (cv && r < Lp && r >= uc) ? __ldg(yc + r) : make_double2(0.0, 0.0);
          }
        };
        load_tile(0);
        for (int tl = 0; tl < ntile; ++tl) {  // one tile per round, eight warps (partials)
          const int slo = __reduce_min_sync(0xffffffffu, uc);
          const bool mt0 = slo <= 7, mt1 = t >= 8;
          // eight independent DMMA chains per warp: [M tile][Vx·Yx, Vy·Yy, Vx·Yy, Vy·Yx]
          double acc[16];
#pragma unroll
          for (int a = 0; a < 16; ++a) acc[a] = 0.0;
#pragma unroll
          for (int i = 0; i < KQ; ++i) {
            const int ks = pp + 8 * i;
            if (ks < nks) {
              const int r = 4 * ks + tq;
              if (mt0) {
                const double2 a = sV[gq * RP + r];
                dmma8x8x4_nv(acc[0], acc[1], a.x, yv[i].x);
                dmma8x8x4_nv(acc[2], acc[3], a.y, yv[i].y);
                dmma8x8x4_nv(acc[4], acc[5], a.x, yv[i].y);
                dmma8x8x4_nv(acc[6], acc[7], a.y, yv[i].x);
              }
              if (mt1) {
                const double2 a = sV[(8 + gq) * RP + r];
                dmma8x8x4_nv(acc[8], acc[9], a.x, yv[i].x);
                dmma8x8x4_nv(acc[10], acc[11], a.y, yv[i].y);
                dmma8x8x4_nv(acc[12], acc[13], a.x, yv[i].y);
                dmma8x8x4_nv(acc[14], acc[15], a.y, yv[i].x);
              }
            }
          }
          // scratch [pp][mt * 4 + product][lane][2]
          double* sc = s_sc + (size_t)(pp * 8) * 64;
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            sc[a * 64 + lane * 2 + 0] = acc[2 * a];
            sc[a * 64 + lane * 2 + 1] = acc[2 * a + 1];
          }
          if (tl + 1 < ntile) load_tile(tl + 1);  // in flight during the combine
          __syncthreads();
          // each product ((P0 + P1) + (P2 + P3)) + ((P4 + P5) + (P6 + P7)); Re d = XX + YY,
          // Im d = XY − YX -> s_d[entry][s]
          {
            const int idx = threadIdx.x;  // 2 x 2 x 64 = 256 outputs
            const int mt = idx >> 7, ri = (idx >> 6) & 1, o = idx & 63;
            const int ln = o >> 1, bb = o & 1;
            const int s = 8 * mt + (ln >> 2), ecol = tl * 8 + 2 * (ln & 3) + bb;
            if (ecol < nch && s <= t) {
              const double* sc0 = s_sc + (size_t)(mt * 4 + 2 * ri) * 64 + o;  // pp stride 512
              auto psum = [&](const double* q) {
                return __dadd_rn(__dadd_rn(__dadd_rn(q[0], q[512]), __dadd_rn(q[1024], q[1536])),
                                 __dadd_rn(__dadd_rn(q[2048], q[2560]), __dadd_rn(q[3072], q[3584])));
              };
              const double p0 = psum(sc0), p1 = psum(sc0 + 64);
              reinterpret_cast<double*>(s_d + ecol * kLazySD + s)[ri] =
                  ri == 0 ? __dadd_rn(p0, p1) : __dsub_rn(p0, p1);
            }
          }
          __syncthreads();
        }
        // phase B: a half-warp per column, lane s <-> panel step s (compact code: a fully
        // unrolled thread-per-column form ran out of the instruction cache): f = M d (d_s of
        // earlier refreshes of this panel from Dd), R(j0+s, c), then the downdates of ν² in s
        // order, identical on the 16 lanes of the column
        for (int e1 = 2 * warp; e1 < nch; e1 += 2 * kLazyWarps) {
          const int hf = lane >> 4, s = lane & 15;
          const int e = e1 + hf;
          const bool ok = e < nch;  // uniform over the half-warp
          const int i = ok ? list[e0 + e] : list[e0 + e1];
          const int64_t c = c_lo + i;
          const int u = ok ? upd_s[i] : kNB;
          double2* yc = Y + c * ldy;
          double2* Fc = w.F + c * kNB;
          double2* Dc = w.Dd + c * kNB;
          const bool mine = ok && s >= u && s <= t;  // this refresh computes step s
          double2 dl = make_double2(0.0, 0.0), fl = dl, yl = dl;
          if (ok && s <= t) {  // F, Dd and these rows of Y are written only by this CTA
            if (s < u) {
              dl = Dc[s];
              fl = Fc[s];
            } else {
              dl = s_d[e * kLazySD + s];
              yl = yc[j0 + s];
            }
          }
          double fr = 0.0, fi = 0.0;
#pragma unroll
          for (int s1 = 0; s1 < kNB; ++s1) {  // f_s = Σ_{s1<=s} M[s][s1] d_s1, ascending
            const double dx = __shfl_sync(0xffffffffu, dl.x, s1, 16);
            const double dy = __shfl_sync(0xffffffffu, dl.y, s1, 16);
            if (mine && s1 <= s) cmac_add(fr, fi, s_M[s][s1], make_double2(dx, dy));
          }
          if (mine) {
            fl = make_double2(fr, fi);
            Fc[s] = fl;
            Dc[s] = dl;
          }
          double rr0 = 0.0, ri0 = 0.0;
#pragma unroll
          for (int s1 = 0; s1 < kNB; ++s1) {  // R = y_s − Σ_{s1<=s} V[j0+s, s1] f_s1, ascending
            const double fx = __shfl_sync(0xffffffffu, fl.x, s1, 16);
            const double fy = __shfl_sync(0xffffffffu, fl.y, s1, 16);
            if (mine && s1 <= s) cmac_add(rr0, ri0, sV[s1 * RP + s], make_double2(fx, fy));
          }
          const double2 Rj = make_double2(__dsub_rn(yl.x, rr0), __dsub_rn(yl.y, ri0));
          const double nu2_0 = ok ? nu_s[i] : 0.0, ref2_0 = ok ? ref_s[i] : 0.0;
          double nu2 = nu2_0, ref2 = ref2_0;
          // fast path: the downdates in s order without a recompute (unrolled; the shuffles do
          // not depend on ν²); if any step of either column would need the exact recompute, both
          // redo their chain in the general loop below (the same arithmetic)
          bool slow = false;
#pragma unroll
          for (int s1 = 0; s1 < kNB; ++s1) {
            const double rx = __shfl_sync(0xffffffffu, Rj.x, s1, 16);
            const double ry = __shfl_sync(0xffffffffu, Rj.y, s1, 16);
            if (ok && s1 >= u && s1 <= t) {
              const double d2 = __fma_rn(-rx, rx, __fma_rn(-ry, ry, nu2));
              slow |= !(nu2 > 0.0) || !(d2 > kRecompTol * ref2);
              nu2 = d2 > 0.0 ? d2 : 0.0;
            }
          }
          slow = __any_sync(0xffffffffu, slow);
          if (slow) {
            nu2 = nu2_0;
            ref2 = ref2_0;
          }
          const int ulo = slow ? min(u, __shfl_xor_sync(0xffffffffu, u, 16)) : t + 1;
          for (int s1 = ulo; s1 <= t; ++s1) {  // ν² ← ν² − |R(j0+s1, c)|²
            const double rx = __shfl_sync(0xffffffffu, Rj.x, s1, 16);
            const double ry = __shfl_sync(0xffffffffu, Rj.y, s1, 16);
            const bool act = ok && s1 >= u;
            const double d2 = __fma_rn(-rx, rx, __fma_rn(-ry, ry, nu2));
            const bool need = act && (!(nu2 > 0.0) || !(d2 > kRecompTol * ref2));
            if (act) nu2 = d2 > 0.0 ? d2 : 0.0;
            if (__any_sync(0xffffffffu, need)) {
              // rare: exact ν² of rows j0+s1+1..l-1 of y^(j0+s1+1) (Y not yet written), the
              // column's 16 lanes over rows s + 16 q
              double nn = 0.0;
              for (int q = 0; q < 2 * qn; ++q) {
                const int r = s + 16 * q;
                const bool in = need && r > s1 && r < Lp;
                double2 z = in ? yc[j0 + r] : make_double2(0.0, 0.0);
                for (int s2 = 0; s2 <= s1; ++s2) {
                  const double fx = __shfl_sync(0xffffffffu, fl.x, s2, 16);
                  const double fy = __shfl_sync(0xffffffffu, fl.y, s2, 16);
                  if (in) cmac_sub(z, sV[s2 * RP + r], make_double2(fx, fy));
                }
                nn = __fma_rn(z.x, z.x, nn);
                nn = __fma_rn(z.y, z.y, nn);
              }
#pragma unroll
              for (int m = 8; m >= 1; m >>= 1) nn = __dadd_rn(nn, __shfl_xor_sync(0xffffffffu, nn, m));
              if (need) nu2 = ref2 = nn;
            }
          }
          if (mine) yc[j0 + s] = Rj;
          if (ok && s == 0) {
            nu_s[i] = nu2;
            ref_s[i] = ref2;
            upd_s[i] = t + 1;
          }
        }
        __syncthreads();
      }
    };

    pass(tau);
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 2] = globaltimer();
    exchange(t + 1);
    // the top two are exact once every column not refreshed at this step has a bound below b2;
    // otherwise refresh down to b2 (or, with fewer than two exact values, the top stale bound)
    while (s_top.m >= 0.0 && !(s_top.b2 > s_top.m)) {
      const double thr = s_top.b2 >= 0.0 ? s_top.b2 : s_top.m;
      if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 7] += 1;
      pass(thr);
      exchange(t + 1);
    }
    if (w.trace && b == 0 && threadIdx.x == 0) w.trace[8 * j + 3] = globaltimer();
  }
  // the norms² go back for the next panel (every column is exact as of step jend)
  for (int i = threadIdx.x; i < ncol; i += kLazyThreads) {
    w.nu[c_lo + i] = nu_s[i];
    w.nuref[c_lo + i] = ref_s[i];
  }
  if (b == 0 && threadIdx.x == 0) sh.w[0].scal[1] = (double)xc;
  if (bl == 0 && threadIdx.x == 0) out.info[1] = jend;
}

size_t qrcp_work_bytes(int64_t n, int64_t l, int max_blocks) {
  return (size_t)2 * n * sizeof(double) + (size_t)2 * 8 * max_blocks * sizeof(double) +
         (size_t)l * kNB * sizeof(double2) + (size_t)2 * kNB * n * sizeof(double2) +
         (size_t)2 * max_blocks * l * sizeof(double2) + 512;
}

QrcpWork qrcp_work_carve(void* buf, int64_t n, int64_t l, int max_blocks) {
  char* p = (char*)buf;
  QrcpWork w{};
  w.max_blocks = max_blocks;
  w.V = (double2*)p;  // 16-byte aligned first
  p += (size_t)l * kNB * sizeof(double2);
  w.F = (double2*)p;
  p += (size_t)kNB * n * sizeof(double2);
  w.Dd = (double2*)p;  // the lazy kernel's d_s(c) of the panel
  p += (size_t)kNB * n * sizeof(double2);
  w.xslot = (double2*)p;
  p += (size_t)2 * max_blocks * l * sizeof(double2);
  w.nu = (double*)p;
  p += (size_t)n * sizeof(double);
  w.nuref = (double*)p;
  p += (size_t)n * sizeof(double);
  w.cand = (double*)p;
  p += (size_t)2 * 8 * max_blocks * sizeof(double);  // 3 (ring) or 8 (lazy: 64-byte records) per CTA
  w.scal = (double*)p;
  p += 64;
  w.bar = (unsigned*)p;
  return w;
}

static int qrcp_blocks(const void* kern, size_t smem, int num_sms, int max_blocks, int64_t n,
                       cudaError_t* err) {
  int occ = 0;
  *err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kQrcpThreads, smem);
  if (*err != cudaSuccess) return 0;
  if (occ < 1) {
    *err = cudaErrorInvalidConfiguration;
    return 0;
  }
  int blocks = num_sms * (occ < 2 ? occ : 2);
  if (blocks > max_blocks) blocks = max_blocks;
  const int64_t min_cols = 8;  // keep >= 8 columns per CTA on small n
  if ((int64_t)blocks * min_cols > n) blocks = (int)((n + min_cols - 1) / min_cols);
  return blocks < 1 ? 1 : blocks;
}

template <int MAXQ>
static cudaError_t launch_qrcp(double2* Y, int64_t ldy, int l, int64_t n, int k, double tol_rel,
                               const QrcpOut& out, const QrcpWork& w, int num_sms,
                               cudaStream_t st, int* launches) {
  const size_t smem = sizeof(double2) * kQB * MAXQ * 32;
  cudaError_t e = ensure_dyn_smem((const void*)k_qrcp<MAXQ>, smem);
  if (e != cudaSuccess) return e;
  const int blocks = qrcp_blocks((const void*)k_qrcp<MAXQ>, smem, num_sms, w.max_blocks, n, &e);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(w.bar, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  QrcpOut o = out;
  QrcpWork ww = w;
  void* args[] = {&Y, &ldy, &l, &n, &k, &tol_rel, &o, &ww};
  *launches += 1;
  return cudaLaunchCooperativeKernel((void*)k_qrcp<MAXQ>, dim3(blocks), dim3(kQrcpThreads), args,
                                     smem, st);
}

// The shared-memory-resident exact kernel, when the columns fit (2 CTAs per SM, else 1);
// cudaErrorNotSupported when they do not (the caller falls back to k_qrcp).
template <int MAXQ>
static cudaError_t launch_qrcp_smem(double2* Y, int64_t ldy, int l, int64_t n, int k,
                                    double tol_rel, const QrcpOut& out, const QrcpWork& w,
                                    int num_sms, cudaStream_t st, int* launches) {
  auto kern = k_qrcp_smem<MAXQ>;
  cudaError_t e;
  // device and function attributes and occupancies: cached per device (rid_host.h; host API
  // calls on every decompose cost ~10 us, a visible share of the small configs' step)
  int optin = 0;
  size_t fstatic = 0;
  if ((e = optin_smem(&optin)) != cudaSuccess) return e;
  if ((e = static_smem((const void*)kern, &fstatic)) != cudaSuccess) return e;
  for (int per_sm = 2; per_sm >= 1; --per_sm) {
    int blocks = num_sms * per_sm;
    if (blocks > w.max_blocks) blocks = w.max_blocks;
    if ((int64_t)blocks * 8 > n) blocks = (int)((n + 7) / 8);
    if (blocks < 1) blocks = 1;
    const int per = (int)((n + blocks - 1) / blocks);
    blocks = (int)((n + per - 1) / per);
    const size_t smem = (size_t)MAXQ * 32 * sizeof(double2) + (size_t)((per + 1) & ~1) * 8 +
                        (size_t)per * l * sizeof(double2);
    const size_t cap = (size_t)optin / per_sm - fstatic - 1024;
    if (smem > cap) continue;
    int occ = 0;
    if ((e = occupancy((const void*)kern, kQrcpThreads, smem, &occ)) != cudaSuccess) return e;
    if (occ * num_sms < blocks) continue;  // a cooperative launch needs every CTA resident
    if ((e = cudaMemsetAsync(w.bar, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    QrcpOut o = out;
    QrcpWork ww = w;
    int perv = per;
    void* args[] = {&Y, &ldy, &l, &n, &k, &tol_rel, &o, &ww, &perv};
    *launches += 1;
    return cudaLaunchCooperativeKernel((void*)kern, dim3(blocks), dim3(kQrcpThreads), args, smem,
                                       st);
  }
  return cudaErrorNotSupported;
}

// The shared-memory-resident exact kernel as ONE cluster of cs CTAs (distributed shared memory
// exchange, cluster barrier; small sketches: C1): cudaErrorNotSupported when the columns do not
// fit (the caller falls back to the grid-wide kernel).
template <int MAXQ>
static cudaError_t launch_qrcp_cluster(double2* Y, int64_t ldy, int l, int64_t n, int k,
                                       double tol_rel, const QrcpOut& out, const QrcpWork& w,
                                       cudaStream_t st, int* launches) {
  auto kern = k_qrcp_smem<MAXQ, true>;
  cudaError_t e;
  int optin = 0;
  size_t fstatic = 0;
  if ((e = optin_smem(&optin)) != cudaSuccess) return e;
  if ((e = static_smem((const void*)kern, &fstatic)) != cudaSuccess) return e;
  if ((e = ensure_func_attr((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed,
                            1)) != cudaSuccess)
    return e;
  for (int cs : {16, 8}) {
    int per = (int)((n + cs - 1) / cs);
    if (per < 1) per = 1;
    const int blocks = (int)((n + per - 1) / per);
    const size_t smem = (size_t)MAXQ * 32 * sizeof(double2) + (size_t)((per + 1) & ~1) * 8 +
                        (size_t)per * l * sizeof(double2) + (size_t)2 * l * sizeof(double2) +
                        6 * sizeof(double);
    if (smem > (size_t)optin - fstatic - 1024) continue;
    if ((e = ensure_dyn_smem((const void*)kern, smem)) != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(kQrcpThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)blocks;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, (const void*)kern, &cfg) != cudaSuccess ||
        clusters < 1) {
      cudaGetLastError();
      continue;
    }
    *launches += 1;
    return cudaLaunchKernelEx(&cfg, kern, Y, ldy, l, n, k, tol_rel, out, w, per);
  }
  return cudaErrorNotSupported;
}

// Panels of nb steps (k_qrcp_ring), each followed by the tensor-core trailing update
// Y[jend:l, :] -= V[jend:l, 0:nb] · F[0:nb, :] (k_zgemm.cu mode 2) of every rank's block.
// The grid is G rank groups of cpr CTAs (G = 1: the whole-sketch QR).

// RID_QRCP_LAZY: 1 the lazy-refresh kernel where it fits (l <= 544), 2 the same kernel
// refreshing every column at every step (bitwise the same results, tested), 0 the ring kernel.
// Default: lazy for l > 384 (C4: 18.5 -> 17.3 ms), the ring kernel below (C5, l = 272: its
// streaming pass over 272 rows is cheaper than the lazy kernel's per-step latency, 7.2 vs 8.1 ms).
static int qrcp_lazy_mode(int l) {
  if (const char* v = select_env("RID_QRCP_LAZY")) {
    const int m = atoi(v);
    return (m == 0 || m == 2) ? m : 1;
  }
  return l > 384 ? 1 : 0;
}

template <int MAXQ>
static cudaError_t launch_qrcp_lazy(const QrShards& sh, int64_t ldy, int l, int k, double tol_rel,
                                    int num_sms, cudaStream_t st, int* launches, int nbw,
                                    int mode) {
  auto kern = k_qrcp_lazy<MAXQ>;
  cudaError_t e;
  const int G = sh.G;
  const int64_t n = sh.n_loc;
  if (G < 1 || G > kQrMaxRanks || n < 1 || l > 32 * MAXQ) return cudaErrorInvalidValue;
  int optin = 0;
  size_t fstatic = 0;
  if ((e = optin_smem(&optin)) != cudaSuccess) return e;
  if ((e = static_smem((const void*)kern, &fstatic)) != cudaSuccess) return e;
  // CTAs per rank: the SMs split evenly over the ranks (one CTA per SM, cooperative); a
  // column's arithmetic does not depend on its CTA, so any split gives the same bits
  int cpr = num_sms / G;
  if (const char* v = experiment_env("RID_QRCP_LAZY_CTAS"))  // CTAs per rank (fewer: cheaper
    if (atoi(v) > 0 && atoi(v) < cpr) cpr = atoi(v);          // exchange, longer passes)
  if ((int64_t)cpr * 8 > n) cpr = (int)((n + 7) / 8);
  if (cpr * G > sh.w[0].max_blocks) cpr = sh.w[0].max_blocks / G;
  if (cpr < 1) cpr = 1;
  const int per = (int)((n + cpr - 1) / cpr);
  cpr = (int)((n + per - 1) / per);
  const int blocks = cpr * G;
  const size_t smem = (size_t)kNB * (32 * MAXQ + 4) * sizeof(double2) +
                      (size_t)kLazyChunk * kLazySD * sizeof(double2) + kLazyScratch * sizeof(double) +
                      (size_t)per * (2 * sizeof(double) + 2 * sizeof(int));
  if (smem + fstatic + 1024 > (size_t)optin) return cudaErrorNotSupported;  // the ring kernel
  if ((e = ensure_dyn_smem((const void*)kern, smem)) != cudaSuccess) return e;
  double kappa = 8.0;  // the refresh threshold's slack (changes no bit of the result, only work;
                       // C4: 3 / 6 / 10 / 20 -> 18.0 / 17.3 / 17.5 / 18.6 ms)
  if (const char* v = select_env("RID_QRCP_KAPPA")) kappa = atof(v);
  for (int g = 0; g < G; ++g) {
    if ((e = cudaMemsetAsync(sh.out[g].info, 0, 2 * sizeof(int), st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(sh.w[g].F, 0, (size_t)kNB * n * sizeof(double2), st)) != cudaSuccess)
      return e;
  }
  for (int j0 = 0; j0 < k; j0 += nbw) {
    const int jend = (j0 + nbw < k) ? j0 + nbw : k;
    if ((e = cudaMemsetAsync(sh.w[0].bar, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    QrShards shv = sh;
    int64_t ldyv = ldy;
    int lv = l, kv = k, j0v = j0, jendv = jend, perv = per, cprv = cpr, modev = mode;
    double tolv = tol_rel, kappav = kappa;
    void* args[] = {&shv, &ldyv, &lv, &kv, &j0v, &jendv, &tolv, &perv, &cprv, &kappav, &modev};
    e = cudaLaunchCooperativeKernel((void*)kern, dim3(blocks), dim3(kLazyThreads), args, smem, st);
    if (e != cudaSuccess) return e;
    *launches += 1;
    if (jend < k) {  // trailing rows jend..l-1 of every column of every rank (as the ring kernel)
      for (int g = 0; g < G; ++g) {
        e = zgemm_ordered(sh.w[g].V + jend, l, sh.w[g].F, kNB, sh.Y[g] + jend, ldy, l - jend, n,
                          jend - j0, 2, 0.0, 0, 0, st);
        if (e != cudaSuccess) return e;
        *launches += 1;
      }
    }
  }
  return cudaSuccess;
}

template <int MAXQ>
static cudaError_t launch_qrcp_blocked(const QrShards& sh, int64_t ldy, int l, int k,
                                       double tol_rel, int num_sms, cudaStream_t st,
                                       int* launches, int nbw) {
  auto kern = k_qrcp_ring<MAXQ>;
  cudaError_t e;
  if constexpr (MAXQ <= 17) {
    const int mode = qrcp_lazy_mode(l);
    if (mode != 0) {
      e = launch_qrcp_lazy<MAXQ>(sh, ldy, l, k, tol_rel, num_sms, st, launches, nbw, mode);
      if (e != cudaErrorNotSupported) return e;
    }
  }
  const int G = sh.G;
  const int64_t n = sh.n_loc;
  if (G < 1 || G > kQrMaxRanks || n < 1) return cudaErrorInvalidValue;
  int optin = 0;  // cached per device (see launch_qrcp_smem)
  size_t fstatic = 0;
  if ((e = optin_smem(&optin)) != cudaSuccess) return e;
  if ((e = static_smem((const void*)kern, &fstatic)) != cudaSuccess) return e;
  // CTAs per rank: the SMs split evenly over the ranks (one CTA per SM, cooperative)
  int cpr = num_sms / G;
  if ((int64_t)cpr * 8 > n) cpr = (int)((n + 7) / 8);
  if (cpr * G > sh.w[0].max_blocks) cpr = sh.w[0].max_blocks / G;
  if (cpr < 1) cpr = 1;
  // columns per CTA: a multiple of 32, so a column's lane in its batch (which rotates the order
  // of its 16 row-partial sums, bank-conflict avoidance) is its global index mod 32 whenever
  // n_loc is a multiple of 32: the same bits for every G
  int per = (int)((n + cpr - 1) / cpr);
  per = (per + 31) / 32 * 32;
  cpr = (int)((n + per - 1) / per);
  const int blocks = cpr * G;
  const size_t fixed = (size_t)kMaxSlots * 8 + (size_t)(MAXQ * 32 + 32) * sizeof(double2) + 128;
  const size_t avail = (size_t)optin - fstatic - 1024;
  const size_t slot_bytes = (size_t)32 * kCH * sizeof(double2);
  if (avail < fixed + 2 * slot_bytes) return cudaErrorInvalidConfiguration;
  int slots = (int)((avail - fixed) / slot_bytes);
  if (slots > kMaxSlots) slots = kMaxSlots;
  // ncw streaming warps with D slots each: D >= 2 keeps a chunk in flight while one is reduced
  // one batch of 32 columns per streaming warp where possible (the critical path of a step is
  // the busiest warp), each with D >= 2 boxes in flight
  const int nbat = (per + 31) / 32;
  int ncw = kRingWarps - 1;
  if (ncw > nbat) ncw = nbat;
  if (ncw > slots / 2) ncw = slots / 2;
  if (const char* v = experiment_env("RID_QRCP_NCW")) {  // experiments
    const int x = atoi(v);
    if (x >= 1 && x <= slots / 2) ncw = x;
  }
  int D = slots / ncw;
  if (D > 4) D = 4;
  if (const char* v = experiment_env("RID_QRCP_D")) {  // ring-depth experiments
    const int x = atoi(v);
    if (x >= 2 && x * ncw <= slots) D = x;
  }
  const size_t smem = fixed + (size_t)ncw * D * slot_bytes;
  if ((e = ensure_dyn_smem((const void*)kern, smem)) != cudaSuccess) return e;
  // 2D tensor map of each rank's block as a (2l doubles) x n_loc matrix, boxes of kCH complex
  // rows x 32 columns
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    if ((e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault,
                                     &qr)) != cudaSuccess)
      return e;
    if (qr != cudaDriverEntryPointSuccess || !encode) return cudaErrorSymbolNotFound;
  }
  RingMaps tm;
  for (int g = 0; g < G; ++g) {
    const cuuint64_t gdim[2] = {(cuuint64_t)(2 * l), (cuuint64_t)n};
    const cuuint64_t gstride[1] = {(cuuint64_t)ldy * sizeof(double2)};
    const cuuint32_t box[2] = {(cuuint32_t)(2 * kCH), 32u};
    const cuuint32_t estr[2] = {1u, 1u};
    if (encode(&tm.m[g], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)sh.Y[g], gdim, gstride, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  for (int g = 0; g < G; ++g) {
    if ((e = cudaMemsetAsync(sh.out[g].info, 0, 2 * sizeof(int), st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(sh.w[g].F, 0, (size_t)kNB * n * sizeof(double2), st)) != cudaSuccess)
      return e;
  }
  for (int j0 = 0; j0 < k; j0 += nbw) {
    const int jend = (j0 + nbw < k) ? j0 + nbw : k;
    if ((e = cudaMemsetAsync(sh.w[0].bar, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    QrShards shv = sh;
    int64_t ldyv = ldy;
    int lv = l, kv = k, j0v = j0, jendv = jend, ncwv = ncw, Dv = D, perv = per, cprv = cpr;
    double tolv = tol_rel;
    double l2_keep = 80.0 * (1 << 20);  // bytes of the trailing block kept in L2 (126 MB L2)
    if (const char* v = experiment_env("RID_QRCP_L2KEEP_MB")) l2_keep = atof(v) * (1 << 20);
    void* args[] = {&shv, &ldyv, &lv, &kv, &j0v, &jendv, &tolv, &ncwv, &Dv, &perv, &cprv,
                    &l2_keep, &tm};
    e = cudaLaunchCooperativeKernel((void*)kern, dim3(blocks), dim3(kRingThreads), args, smem, st);
    if (e != cudaSuccess) return e;
    *launches += 1;
    if (jend < k) {  // trailing rows jend..l-1 of every column of every rank
      // (a CUDA-core version holding V in registers was measured no faster: 2.97 vs 2.94 ms of
      // updates at C4, both ≈3 TB/s — the update has 4 flop/B against a 5.7 flop/B FP64 ridge)
      for (int g = 0; g < G; ++g) {
        e = zgemm_ordered(sh.w[g].V + jend, l, sh.w[g].F, kNB, sh.Y[g] + jend, ldy, l - jend, n,
                          jend - j0, 2, 0.0, 0, 0, st);
        if (e != cudaSuccess) return e;
        *launches += 1;
      }
    }
  }
  return cudaSuccess;
}

static int blocked_panel_width() {
  int nbw = kNBDefault;
  if (const char* v = select_env("RID_QRCP_NB")) nbw = atoi(v);  // tested: J, P independent of nb
  if (nbw < 1 || nbw > kNB) nbw = kNBDefault;
  return nbw;
}

static QrShards one_shard(double2* Y, int64_t n, const QrcpOut& out, const QrcpWork& w) {
  QrShards sh;
  sh.G = 1;
  sh.n_loc = n;
  sh.Y[0] = Y;
  sh.out[0] = out;
  sh.w[0] = w;
  return sh;
}

cudaError_t qrcp_sharded(const QrShards& sh, int64_t ldy, int64_t l, int64_t k, double tol_rel,
                         int num_sms, cudaStream_t st, int* launches) {
  int dummy = 0;
  if (!launches) launches = &dummy;
  if (sh.G < 1 || sh.G > kQrMaxRanks || sh.n_loc < 1 || k < 1 || k > l ||
      k > (int64_t)sh.G * sh.n_loc)
    return cudaErrorInvalidValue;
  const int li = (int)l, ki = (int)k, nbw = blocked_panel_width();
  const int qneed = (li + 31) / 32;
#define RID_QS(QV) \
  if (qneed <= QV) return launch_qrcp_blocked<QV>(sh, ldy, li, ki, tol_rel, num_sms, st, launches, nbw);
  RID_QS(1) RID_QS(2) RID_QS(3) RID_QS(4) RID_QS(5) RID_QS(6) RID_QS(8) RID_QS(9) RID_QS(12)
  RID_QS(17) RID_QS(24) RID_QS(32) RID_QS(48) RID_QS(64)
#undef RID_QS
  return cudaErrorInvalidValue;  // l > 2048 unsupported
}

cudaError_t qrcp(double2* Y, int64_t ldy, int64_t l, int64_t n, int64_t k, double tol_rel,
                 const QrcpOut& out, const QrcpWork& w, int num_sms, cudaStream_t st,
                 int* launches, int variant) {
  const int li = (int)l, ki = (int)k;
  const int qneed = (li + 31) / 32;
  // Blocked panels pay off once the sketch no longer fits in L2 (C4: 34.2 -> 21.1 ms, C5: 9.2 ->
  // 6.6 ms); small sketches (C2/C3, ~10 MB) are latency-bound and the single persistent kernel
  // is faster there (C2: 0.68 vs 1.04 ms). Measured on B200, tools/trace_qrcp.py.
  // variant 0 (small sketches): the one-cluster kernel when the sketch fits in 16 (8) CTAs'
  // shared memory (C1), else the grid-wide shared-memory kernel, else the global-memory one;
  // 3 forces the cluster kernel, 4 the grid-wide shared-memory kernel (tests)
  if (variant < 0) {
    variant = (16.0 * (double)l * (double)n >= 64.0 * (1 << 20)) ? 1 : 0;
    if (const char* v = select_env("RID_QRCP_VARIANT")) variant = atoi(v);
  }
  const int nbw = blocked_panel_width();
  int dummy = 0;
  if (!launches) launches = &dummy;
#define RID_Q(QV)                                                                              \
  if (qneed <= QV) {                                                                           \
    if (variant == 1)                                                                          \
      return launch_qrcp_blocked<QV>(one_shard(Y, n, out, w), ldy, li, ki, tol_rel, num_sms,   \
                                     st, launches, nbw);                                       \
    if (variant == 0 || variant == 3) {                                                        \
      const cudaError_t ec =                                                                   \
          launch_qrcp_cluster<QV>(Y, ldy, li, n, ki, tol_rel, out, w, st, launches);           \
      if (ec != cudaErrorNotSupported || variant == 3) return ec;                              \
    }                                                                                          \
    if (variant == 0 || variant == 4) {                                                        \
      const cudaError_t es =                                                                   \
          launch_qrcp_smem<QV>(Y, ldy, li, n, ki, tol_rel, out, w, num_sms, st, launches);     \
      if (es != cudaErrorNotSupported) return es;                                              \
    }                                                                                          \
    return launch_qrcp<QV>(Y, ldy, li, n, ki, tol_rel, out, w, num_sms, st, launches);         \
  }
  RID_Q(1) RID_Q(2) RID_Q(3) RID_Q(4) RID_Q(5) RID_Q(6) RID_Q(8) RID_Q(9) RID_Q(12) RID_Q(17)
  RID_Q(24) RID_Q(32)
#undef RID_Q
  // l up to 2048 (the paper's l = 2k with k = 1000): blocked panels only (the exact kernel holds
  // a column segment in registers)
  if (qneed <= 48)
    return launch_qrcp_blocked<48>(one_shard(Y, n, out, w), ldy, li, ki, tol_rel, num_sms, st,
                                   launches, nbw);
  if (qneed <= 64)
    return launch_qrcp_blocked<64>(one_shard(Y, n, out, w), ldy, li, ki, tol_rel, num_sms, st,
                                   launches, nbw);
  return cudaErrorInvalidValue;  // l > 2048 unsupported
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

// The same back-substitutions with one WARP per column of R11^{-1} and the right-hand side in
// registers (lane L holds rows L, L + 32, ...): no CTA barrier per step, and the next step's column
// of R11 is loaded into registers while the current step computes, so a step costs a division, a
// shuffle and the fmas instead of two __syncthreads and an exposed L2 load. Every element sees the
// same fma sequence in the same order as k_tri_inverse: bit-identical (tested).
template <int NSLOT>
__global__ void __launch_bounds__(256) k_tri_inverse_warp(const double2* __restrict__ R11, int k,
                                                          double2* __restrict__ Rinv) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= k) return;  // warp-uniform
  double2 b[NSLOT], rcur[NSLOT], rnext[NSLOT];
#pragma unroll
  for (int q = 0; q < NSLOT; ++q) {
    b[q] = make_double2((32 * q + lane == c) ? 1.0 : 0.0, 0.0);
    rcur[q] = make_double2(0.0, 0.0);
    rnext[q] = make_double2(0.0, 0.0);
  }
  // column c of R11 (rows above the diagonal) and its diagonal: the first step's operands
  double dcur = __ldg(&R11[(int64_t)c * k + c].x);
#pragma unroll
  for (int q = 0; q < NSLOT; ++q) {
    const int i = 32 * q + lane;
    if (i < c) rcur[q] = __ldg(R11 + (int64_t)c * k + i);
  }
#pragma unroll
  for (int q = NSLOT - 1; q >= 0; --q) {
    if (32 * q > c) continue;
    for (int p = (c - 32 * q < 31 ? c - 32 * q : 31); p >= 0; --p) {
      const int s = 32 * q + p;
      // prefetch column s - 1 (rows < s - 1) and its diagonal
      double dnext = 1.0;
      if (s > 0) {
        dnext = __ldg(&R11[(int64_t)(s - 1) * k + (s - 1)].x);
#pragma unroll
        for (int qq = 0; qq <= q; ++qq) {
          const int i = 32 * qq + lane;
          rnext[qq] = (i < s - 1) ? __ldg(R11 + (int64_t)(s - 1) * k + i) : make_double2(0.0, 0.0);
        }
      }
      const double2 bs = make_double2(__shfl_sync(0xffffffffu, b[q].x, p),
                                       __shfl_sync(0xffffffffu, b[q].y, p));
      const double2 xs = make_double2(__ddiv_rn(bs.x, dcur), __ddiv_rn(bs.y, dcur));
#pragma unroll
      for (int qq = 0; qq < q; ++qq) {
        const double2 r = rcur[qq];
        double2 bi = b[qq];
        bi.x = __fma_rn(-r.x, xs.x, __fma_rn(r.y, xs.y, bi.x));
        bi.y = __fma_rn(-r.x, xs.y, __fma_rn(-r.y, xs.x, bi.y));
        b[qq] = bi;
      }
      if (lane < p) {
        const double2 r = rcur[q];
        double2 bi = b[q];
        bi.x = __fma_rn(-r.x, xs.x, __fma_rn(r.y, xs.y, bi.x));
        bi.y = __fma_rn(-r.x, xs.y, __fma_rn(-r.y, xs.x, bi.y));
        b[q] = bi;
      } else if (lane == p) {
        b[q] = xs;
      }
#pragma unroll
      for (int qq = 0; qq <= q; ++qq) rcur[qq] = rnext[qq];
      dcur = dnext;
    }
  }
#pragma unroll
  for (int q = 0; q < NSLOT; ++q) {
    const int i = 32 * q + lane;
    if (i < k) Rinv[(int64_t)c * k + i] = (i <= c) ? b[q] : make_double2(0.0, 0.0);
  }
}

cudaError_t tri_inverse(const double2* R11, int64_t k, double2* Rinv, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  const char* old = select_env("RID_TRI_OLD");
  if (!(old && atoi(old) != 0) && k <= 512) {  // k > 512: 32+ slots per lane would spill
    const unsigned g = (unsigned)((k + 7) / 8);
    if (k <= 64) k_tri_inverse_warp<2><<<g, 256, 0, st>>>(R11, (int)k, Rinv);
    else if (k <= 128) k_tri_inverse_warp<4><<<g, 256, 0, st>>>(R11, (int)k, Rinv);
    else if (k <= 256) k_tri_inverse_warp<8><<<g, 256, 0, st>>>(R11, (int)k, Rinv);
    else k_tri_inverse_warp<16><<<g, 256, 0, st>>>(R11, (int)k, Rinv);
    return cudaGetLastError();
  }
  const size_t sm = (size_t)k * sizeof(double2);
  if (sm > 48 * 1024) {
    cudaError_t e = ensure_dyn_smem((const void*)k_tri_inverse, sm);
    if (e != cudaSuccess) return e;
  }
  k_tri_inverse<<<(unsigned)k, 256, sm, st>>>(R11, (int)k, Rinv);
  return cudaGetLastError();
}

}  // namespace rid
