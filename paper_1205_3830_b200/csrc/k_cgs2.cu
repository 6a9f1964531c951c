// k_cgs2.cu — the paper's own QR of the sketch: column-pivoted classical
// Gram-Schmidt "with iteration" (§3.2: one reorthogonalisation pass, "twice is
// enough"), the greedy column choice of PAPER.md:82-86 (§2, Eqs. 8–9), on the GPU.
//
// Step j (the order of oracle/rid_oracle.c orc_pivoted_cgs2, which follows the paper):
//   1. nu_c = ||W_c|| exactly for every unchosen column (reading R11), p = argmax, ties -> lowest
//      index (R8); rank failure when nu_p < 1e-13 max_c ||Y_c|| (R13);
//   2. q = W_p, twice: coef = Q_j^H q (all from the same q: classical), q -= Q_j coef;
//   3. q_j = q / ||q||;
//   4. W_c -= q_j (q_j^H W_c) for every unchosen column.
// After k steps R = Q^H Y (k x n, original column order) on the tensor-core GEMM, as the oracle
// forms it. W is a copy of Y (it keeps all l rows: unlike Householder nothing shrinks, which is
// the paper's own remark that Householder "should result in similar stability with only half
// the runtime").
//
// Kernels per step: k_cgs_project (steps 4 of j-1 and 1 of j fused: one read-modify-write pass
// over W, warp per column, the last CTA to finish reduces the per-CTA (best, second, index)
// candidates), then k_cgs_coef / k_cgs_update twice (step 2; q and Q stay L2-resident).
// Everything after a rank failure is a no-op (the flag lives in device memory; no host sync).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "rid_internal.h"

namespace rid {
namespace {

constexpr int kProjThreads = 256;  // 8 warps, warp per column
constexpr int kUpdWarps = 16;      // k_cgs_update: 32 rows x 16 warps splitting the t range

struct CgsState {
  int64_t p;        // the pivot of the current step
  int fail;         // rank failure seen: every later kernel returns at once
  unsigned count;   // last-CTA-done counter of k_cgs_project
  double nu0max;    // max_c ||Y_c|| (the rank threshold's scale)
};

struct Top2 {
  double best, second;
  int64_t idx;
};

__device__ __forceinline__ Top2 top2_empty() { return Top2{-1.0, -1.0, INT64_MAX}; }

// merge two candidate triples: larger value wins, equal values -> lower index (reading R8);
// second = the largest value not taken as best (equal values give margin 0, as the oracle's scan)
__device__ __forceinline__ Top2 top2_merge(const Top2& a, const Top2& b) {
  const bool a_wins = a.best > b.best || (a.best == b.best && a.idx < b.idx);
  Top2 r;
  if (a_wins) {
    r.best = a.best;
    r.idx = a.idx;
    r.second = fmax(a.second, b.best);
  } else {
    r.best = b.best;
    r.idx = b.idx;
    r.second = fmax(b.second, a.best);
  }
  return r;
}

__device__ __forceinline__ Top2 top2_warp(Top2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Top2 u;
    u.best = __shfl_xor_sync(0xffffffffu, v.best, o);
    u.second = __shfl_xor_sync(0xffffffffu, v.second, o);
    u.idx = __shfl_xor_sync(0xffffffffu, v.idx, o);
    v = top2_merge(v, u);
  }
  return v;
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Step 3 of step j-1 (normalise q into Q[:, j-1] and Qh[j-1, :]), step 4 of step j-1 (project
// q_{j-1} out of every unchosen column) and step 1 of step j (exact norms, argmax). j == 0: norms
// of Y only. j == k: normalisation only (one CTA).
__global__ void __launch_bounds__(kProjThreads)
    k_cgs_project(double2* __restrict__ W, int64_t ldw, int64_t l, int64_t n,
                  const double2* __restrict__ qbuf, double2* __restrict__ Q, int64_t ldq,
                  double2* __restrict__ Qh, int64_t ldqh, int64_t j, int64_t k, double tol_rel,
                  unsigned char* __restrict__ chosen, CgsState* __restrict__ st,
                  Top2* __restrict__ cand, int64_t* __restrict__ J, double* __restrict__ resid,
                  double* __restrict__ margin, int* __restrict__ info) {
  extern __shared__ double2 sq[];  // l: q_{j-1}, normalised
  __shared__ double s_red[kProjThreads / 32];
  __shared__ Top2 s_cand[kProjThreads / 32];
  __shared__ bool s_last;
  if (*(volatile int*)&st->fail) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool proj = j > 0;
  const int64_t pprev = proj ? *(volatile int64_t*)&st->p : -1;
  if (proj) {
    double s = 0.0;
    for (int64_t r = tid; r < l; r += kProjThreads) {
      const double2 q = qbuf[r];
      sq[r] = q;
      s += q.x * q.x + q.y * q.y;
    }
    s = warp_sum(s);
    if (lane == 0) s_red[warp] = s;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kProjThreads / 32; ++w) t += s_red[w];
    const double qn = sqrt(t);
    for (int64_t r = tid; r < l; r += kProjThreads) sq[r] = make_double2(sq[r].x / qn, sq[r].y / qn);
    __syncthreads();
    if (blockIdx.x == 0) {
      for (int64_t r = tid; r < l; r += kProjThreads) {
        const double2 q = sq[r];
        Q[(j - 1) * ldq + r] = q;
        Qh[r * ldqh + (j - 1)] = make_double2(q.x, -q.y);
      }
      if (tid == 0) chosen[pprev] = 1;
    }
  }
  if (j >= k) return;
  Top2 mine = top2_empty();
  for (int64_t c = (int64_t)blockIdx.x * (kProjThreads / 32) + warp; c < n;
       c += (int64_t)gridDim.x * (kProjThreads / 32)) {
    if (c == pprev || chosen[c]) continue;
    double2* w = W + c * ldw;
    double s = 0.0;
    if (proj) {
      double ar = 0.0, ai = 0.0;  // q^H w
      for (int64_t r = lane; r < l; r += 32) {
        const double2 x = w[r], q = sq[r];
        ar += q.x * x.x + q.y * x.y;
        ai += q.x * x.y - q.y * x.x;
      }
      ar = warp_sum(ar);
      ai = warp_sum(ai);
      for (int64_t r = lane; r < l; r += 32) {
        double2 x = w[r];
        const double2 q = sq[r];
        x.x -= q.x * ar - q.y * ai;
        x.y -= q.x * ai + q.y * ar;
        w[r] = x;
        s += x.x * x.x + x.y * x.y;
      }
    } else {
      for (int64_t r = lane; r < l; r += 32) {
        const double2 x = w[r];
        s += x.x * x.x + x.y * x.y;
      }
    }
    s = warp_sum(s);
    const Top2 v{sqrt(s), -1.0, c};
    mine = top2_merge(mine, v);
  }
  if (lane == 0) s_cand[warp] = mine;
  __syncthreads();
  if (tid == 0) {
    Top2 b = s_cand[0];
    for (int w = 1; w < kProjThreads / 32; ++w) b = top2_merge(b, s_cand[w]);
    cand[blockIdx.x] = b;
    __threadfence();
    s_last = atomicAdd(&st->count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || warp != 0) return;
  __threadfence();
  Top2 b = top2_empty();
  for (int i = lane; i < (int)gridDim.x; i += 32) {
    Top2 u;
    u.best = __ldcg(&cand[i].best);
    u.second = __ldcg(&cand[i].second);
    u.idx = __ldcg(&cand[i].idx);
    b = top2_merge(b, u);
  }
  b = top2_warp(b);
  if (lane == 0) {
    st->count = 0;
    if (j == 0) st->nu0max = b.best;
    const double nu0max = j == 0 ? b.best : st->nu0max;
    resid[j] = b.best;
    margin[j] = b.second < 0.0 ? __longlong_as_double(0x7ff0000000000000LL)
                               : (b.best - b.second) / b.best;
    if (!(b.best >= tol_rel * nu0max) || b.best == 0.0) {  // reading R13
      st->fail = 1;
      info[0] = 2;
      info[1] = (int)j;
    } else {
      st->p = b.idx;
      J[j] = b.idx;
      info[1] = (int)(j + 1);
    }
  }
}

// coef[t] = Q[:, t]^H q for t < j (warp per t); q = W[:, p] on the first pass, qbuf on the second
__global__ void __launch_bounds__(256)
    k_cgs_coef(const double2* __restrict__ Q, int64_t ldq, int64_t l, int64_t j,
               const double2* __restrict__ W, int64_t ldw, const double2* __restrict__ qbuf,
               int pass, const CgsState* __restrict__ st, double2* __restrict__ coef) {
  if (*(volatile const int*)&st->fail) return;
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= j) return;
  const double2* q = pass == 0 ? W + (*(volatile const int64_t*)&st->p) * ldw : qbuf;
  const double2* qt = Q + t * ldq;
  double cr = 0.0, ci = 0.0;
  for (int64_t r = lane; r < l; r += 32) {
    const double2 a = qt[r], x = q[r];
    cr += a.x * x.x + a.y * x.y;
    ci += a.x * x.y - a.y * x.x;
  }
  cr = warp_sum(cr);
  ci = warp_sum(ci);
  if (lane == 0) coef[t] = make_double2(cr, ci);
}

// qbuf[r] = q[r] - sum_{t<j} Q[r, t] coef[t]  (32 rows per CTA, the t range split over warps)
__global__ void __launch_bounds__(32 * kUpdWarps)
    k_cgs_update(const double2* __restrict__ Q, int64_t ldq, int64_t l, int64_t j,
                 const double2* __restrict__ W, int64_t ldw, double2* qbuf, int pass,
                 const CgsState* __restrict__ st, const double2* __restrict__ coef) {
  extern __shared__ double2 scoef[];  // j
  __shared__ double2 s_part[kUpdWarps][32];
  if (*(volatile const int*)&st->fail) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t t = threadIdx.x; t < j; t += blockDim.x) scoef[t] = coef[t];
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * 32 + lane;
  double sr = 0.0, si = 0.0;
  if (r < l) {
    for (int64_t t = warp; t < j; t += kUpdWarps) {
      const double2 a = Q[t * ldq + r], c = scoef[t];
      sr += a.x * c.x - a.y * c.y;
      si += a.x * c.y + a.y * c.x;
    }
  }
  s_part[warp][lane] = make_double2(sr, si);
  __syncthreads();
  if (warp != 0 || r >= l) return;
  double tr = 0.0, ti = 0.0;
  for (int w = 0; w < kUpdWarps; ++w) {
    tr += s_part[w][lane].x;
    ti += s_part[w][lane].y;
  }
  const double2* q = pass == 0 ? W + (*(volatile const int64_t*)&st->p) * ldw : qbuf;
  const double2 x = q[r];
  qbuf[r] = make_double2(x.x - tr, x.y - ti);
}

// R11[t, s] = R[t, J[s]] for t <= s (column s = step s; the diagonal's real part, its imaginary
// part being rounding: q_s^H Y_{J[s]} is real in exact arithmetic), beta[s] = Re R[s, J[s]]
__global__ void k_cgs_r11(const double2* __restrict__ R, int64_t ldr, const int64_t* __restrict__ J,
                          int64_t k, double2* __restrict__ R11, double* __restrict__ beta) {
  const int64_t s = blockIdx.x;
  const double2* col = R + J[s] * ldr;
  for (int64_t t = threadIdx.x; t <= s; t += blockDim.x) {
    const double2 v = col[t];
    R11[s * k + t] = t == s ? make_double2(v.x, 0.0) : v;
    if (t == s) beta[s] = v.x;
  }
}


// ---------------------------------------------------------------------------------------------
// The same algorithm as one cooperative persistent kernel: per step five grid
// barriers instead of five launches, and each warp's columns are held in registers (NR complex
// per lane) between the q^H w reduction and the update, so a step's W traffic is one read and one
// write with NR loads in flight per lane (l <= 544; longer columns take two passes in chunks, the
// second from L2). Phases of step j (every CTA holds p_j):
//   coef0: coef[t] = Q_t^H W_p (warp per t)                      | barrier
//   upd0:  qbuf = W_p - Q coef (CTA per 32 rows, warps split t)  | barrier
//   coef1, upd1 on qbuf                                          | barrier x2
//   every CTA: q_j = qbuf / ||qbuf|| into shared memory (CTA 0 stores Q, Qh); project q_j out
//   of its warps' columns, exact norms, per-CTA candidate         | barrier
//   every CTA reduces all candidates to p_{j+1} (same order, same bits).
// Every global load here is ld.global.cg (L2): W_p, Q, coef, qbuf, the candidates and the chosen
// flags are written by other CTAs between grid barriers, and L1 is not coherent across SMs.
// ---------------------------------------------------------------------------------------------
struct Cgs2Args {
  double2* W;
  int64_t l, n, k;
  double2* Q;     // l x k (ld l)
  double2* Qh;    // k x l (ld k)
  double2* qbuf;  // l
  double2* coef;  // k
  Top2* cand;     // gridDim.x
  unsigned char* chosen;
  unsigned* bar;
  double tol_rel;
  QrcpOut out;
  int opt;                    // bit 0: alternate the column order per step (RID_CGS2_OPT)
  unsigned long long* trace;  // optional: 8 %globaltimer stamps per step (CTA 0; RID_QRCP_TRACE)
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier: the CTA's writes are ordered before thread 0's arrival by bar.sync, the arrival is
// a gpu-scope release reduction, the wait a gpu-scope acquire load (no full fences; the polling
// is unslept: one thread per CTA on one L2 line)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    while (ld_acquire_u32(bar) < target) {
    }
  }
  __syncthreads();
}

// all CTAs: merge the per-CTA candidates in index order (identical bits everywhere)
__device__ __forceinline__ Top2 reduce_cands(const Top2* cand, int nb, Top2* s_out) {
  if (threadIdx.x < 32) {
    Top2 b = top2_empty();
    for (int i = threadIdx.x; i < nb; i += 32) {
      Top2 u;
      u.best = __ldcg(&cand[i].best);
      u.second = __ldcg(&cand[i].second);
      u.idx = __ldcg(&cand[i].idx);
      b = top2_merge(b, u);
    }
    b = top2_warp(b);
    if (threadIdx.x == 0) *s_out = b;
  }
  __syncthreads();
  return *s_out;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int NR>
__global__ void __launch_bounds__(kProjThreads, 2) k_cgs2_fused(Cgs2Args a) {
  extern __shared__ double2 sq[];  // l: the normalised q_j
  __shared__ Top2 s_cand[kProjThreads / 32];
  __shared__ Top2 s_top;
  __shared__ double s_red[kProjThreads / 32];
  __shared__ double2 s_part[kProjThreads / 32][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = gridDim.x;
  const int64_t gw = (int64_t)blockIdx.x * (kProjThreads / 32) + warp;
  const int64_t nw = (int64_t)nb * (kProjThreads / 32);
  const int64_t l = a.l, n = a.n, k = a.k;
  double2* __restrict__ W = a.W;
  unsigned phase = 0;
  auto barrier = [&]() { grid_sync(a.bar, (unsigned)nb * (++phase)); };
  const bool tr = a.trace && blockIdx.x == 0 && threadIdx.x == 0;
  auto stamp = [&](int64_t j, int q) {
    if (tr) a.trace[8 * j + q] = gtimer();
  };
  // candidates of this CTA -> cand[blockIdx.x]; barrier; reduce; CTA 0 records step j
  auto choose = [&](Top2 mine, int64_t j, double& nu0max) -> Top2 {
    if (lane == 0) s_cand[warp] = mine;
    __syncthreads();
    if (tid == 0) {
      Top2 b = s_cand[0];
      for (int w = 1; w < kProjThreads / 32; ++w) b = top2_merge(b, s_cand[w]);
      a.cand[blockIdx.x] = b;
    }
    barrier();
    const Top2 t = reduce_cands(a.cand, nb, &s_top);
    if (j == 0) nu0max = t.best;
    if (blockIdx.x == 0 && tid == 0) {
      a.out.resid[j] = t.best;
      a.out.margin[j] = t.second < 0.0 ? __longlong_as_double(0x7ff0000000000000LL)
                                       : (t.best - t.second) / t.best;
      if (!(t.best >= a.tol_rel * nu0max) || t.best == 0.0) {  // reading R13
        a.out.info[0] = 2;
        a.out.info[1] = (int)j;
      } else {
        a.out.J[j] = t.idx;
        a.out.info[1] = (int)(j + 1);
      }
    }
    return t;
  };
  double nu0max = 0.0;
  // step 0: norms of Y
  Top2 mine = top2_empty();
  for (int64_t c = gw; c < n; c += nw) {
    const double2* w = W + c * l;
    double s = 0.0;
    for (int64_t r0 = 0; r0 < l; r0 += 32 * NR) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int64_t r = r0 + lane + 32 * i;
        if (r < l) {
          const double2 x = __ldcg(&w[r]);
          s += x.x * x.x + x.y * x.y;
        }
      }
    }
    s = warp_sum(s);
    mine = top2_merge(mine, Top2{sqrt(s), -1.0, c});
  }
  Top2 t = choose(mine, 0, nu0max);
  for (int64_t j = 0; j < k; ++j) {
    if (!(t.best >= a.tol_rel * nu0max) || t.best == 0.0) return;  // same decision in every CTA
    const int64_t p = t.idx;
    const double2* wp = W + p * l;
    stamp(j, 0);
    if (j > 0) {
      for (int pass = 0; pass < 2; ++pass) {
        const double2* qin = pass == 0 ? wp : a.qbuf;
        for (int64_t tt = gw; tt < j; tt += nw) {  // coef
          const double2* qt = a.Q + tt * l;
          double cr = 0.0, ci = 0.0;
          for (int64_t r0 = 0; r0 < l; r0 += 32 * NR) {
#pragma unroll
            for (int i = 0; i < NR; ++i) {
              const int64_t r = r0 + lane + 32 * i;
              if (r < l) {
                const double2 u = __ldcg(&qt[r]), x = __ldcg(&qin[r]);
                cr += u.x * x.x + u.y * x.y;
                ci += u.x * x.y - u.y * x.x;
              }
            }
          }
          cr = warp_sum(cr);
          ci = warp_sum(ci);
          if (lane == 0) a.coef[tt] = make_double2(cr, ci);
        }
        barrier();
        stamp(j, 1 + 2 * pass);
        for (int64_t rb = blockIdx.x; rb * 32 < l; rb += nb) {  // update
          const int64_t r = rb * 32 + lane;
          double sr = 0.0, si = 0.0;
          if (r < l) {
#pragma unroll 8
            for (int64_t tt = warp; tt < j; tt += kProjThreads / 32) {
              const double2 u = __ldcg(&a.Q[tt * l + r]), c = __ldcg(&a.coef[tt]);
              sr += u.x * c.x - u.y * c.y;
              si += u.x * c.y + u.y * c.x;
            }
          }
          s_part[warp][lane] = make_double2(sr, si);
          __syncthreads();
          if (warp == 0 && r < l) {
            double tr = 0.0, ti = 0.0;
            for (int w = 0; w < kProjThreads / 32; ++w) {
              tr += s_part[w][lane].x;
              ti += s_part[w][lane].y;
            }
            const double2 x = __ldcg(&qin[r]);
            a.qbuf[r] = make_double2(x.x - tr, x.y - ti);
          }
          __syncthreads();
        }
        barrier();
        stamp(j, 2 + 2 * pass);
      }
    }
    // q_j = q / ||q|| (q = W_p at step 0), in every CTA
    {
      const double2* qsrc = j > 0 ? a.qbuf : wp;
      double s = 0.0;
      for (int64_t r = tid; r < l; r += kProjThreads) {
        const double2 q = __ldcg(&qsrc[r]);
        sq[r] = q;
        s += q.x * q.x + q.y * q.y;
      }
      s = warp_sum(s);
      if (lane == 0) s_red[warp] = s;
      __syncthreads();
      double tot = 0.0;
      for (int w = 0; w < kProjThreads / 32; ++w) tot += s_red[w];
      const double qn = sqrt(tot);
      for (int64_t r = tid; r < l; r += kProjThreads) sq[r] = make_double2(sq[r].x / qn, sq[r].y / qn);
      __syncthreads();
      if (blockIdx.x == 0) {
        for (int64_t r = tid; r < l; r += kProjThreads) {
          const double2 q = sq[r];
          a.Q[j * l + r] = q;
          a.Qh[r * k + j] = make_double2(q.x, -q.y);
        }
        if (tid == 0) a.chosen[p] = 1;
      }
    }
    stamp(j, 5);
    if (j + 1 == k) return;
    // project q_j out of this warp's unchosen columns; exact norms. Odd steps walk the columns
    // backwards so a step starts on what the previous one left in L2 (read and, still dirty,
    // rewritten there): C4 58.9 -> 54.7 ms. (An L2 prefetch of the warp's next column made it
    // worse, 60.9 ms: the projection got uneven across CTAs.)
    mine = top2_empty();
    const int64_t cnt = gw < n ? (n - 1 - gw) / nw + 1 : 0;
    const bool rev = (a.opt & 1) && (j & 1) != 0;
    for (int64_t ii = 0; ii < cnt; ++ii) {
      const int64_t ci = rev ? cnt - 1 - ii : ii;
      const int64_t c = gw + ci * nw;
      if (c == p || __ldcg(&a.chosen[c])) continue;
      double2* w = W + c * l;
      if (l > 32 * NR) {  // long columns (l > 544): two passes in NR-row chunks, the second from L2
        double ar = 0.0, ai = 0.0;
        for (int64_t r0 = 0; r0 < l; r0 += 32 * NR) {
#pragma unroll
          for (int i = 0; i < NR; ++i) {
            const int64_t r = r0 + lane + 32 * i;
            if (r < l) {
              const double2 x = __ldcg(&w[r]), q = sq[r];
              ar += q.x * x.x + q.y * x.y;
              ai += q.x * x.y - q.y * x.x;
            }
          }
        }
        ar = warp_sum(ar);
        ai = warp_sum(ai);
        double s = 0.0;
        for (int64_t r0 = 0; r0 < l; r0 += 32 * NR) {
#pragma unroll
          for (int i = 0; i < NR; ++i) {
            const int64_t r = r0 + lane + 32 * i;
            if (r < l) {
              double2 x = __ldcg(&w[r]);
              const double2 q = sq[r];
              x.x -= q.x * ar - q.y * ai;
              x.y -= q.x * ai + q.y * ar;
              w[r] = x;
              s += x.x * x.x + x.y * x.y;
            }
          }
        }
        s = warp_sum(s);
        mine = top2_merge(mine, Top2{sqrt(s), -1.0, c});
        continue;
      }
      double2 x[NR];
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int64_t r = lane + 32 * i;
        x[i] = r < l ? __ldcg(&w[r]) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int64_t r = lane + 32 * i;
        if (r < l) {
          const double2 q = sq[r];
          ar += q.x * x[i].x + q.y * x[i].y;
          ai += q.x * x[i].y - q.y * x[i].x;
        }
      }
      ar = warp_sum(ar);
      ai = warp_sum(ai);
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int64_t r = lane + 32 * i;
        if (r < l) {
          const double2 q = sq[r];
          x[i].x -= q.x * ar - q.y * ai;
          x[i].y -= q.x * ai + q.y * ar;
          w[r] = x[i];
          s += x[i].x * x[i].x + x[i].y * x[i].y;
        }
      }
      s = warp_sum(s);
      mine = top2_merge(mine, Top2{sqrt(s), -1.0, c});
    }
    stamp(j, 6);
    t = choose(mine, j + 1, nu0max);
    stamp(j, 7);
  }
}

template <int NR>
cudaError_t launch_fused(const Cgs2Args& a, int num_sms, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (size_t)a.l;
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cgs2_fused<NR>,
                                                                kProjThreads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorNotSupported;
  int blocks = std::min(occ, 2) * num_sms;
  const int64_t need = (a.n + kProjThreads / 32 - 1) / (kProjThreads / 32);
  if (blocks > need) blocks = (int)std::max<int64_t>(need, (a.l + 31) / 32);
  if (blocks < 1) blocks = 1;
  if ((e = cudaMemsetAsync(a.bar, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
  Cgs2Args aa = a;
  void* args[] = {&aa};
  return cudaLaunchCooperativeKernel((void*)k_cgs2_fused<NR>, dim3(blocks), dim3(kProjThreads),
                                     args, smem, st);
}

cudaError_t cgs2_fused(const Cgs2Args& a, int num_sms, cudaStream_t st) {
  const int64_t nr = (a.l + 31) / 32;
  if (nr <= 1) return launch_fused<1>(a, num_sms, st);
  if (nr <= 2) return launch_fused<2>(a, num_sms, st);
  if (nr <= 3) return launch_fused<3>(a, num_sms, st);
  if (nr <= 5) return launch_fused<5>(a, num_sms, st);
  if (nr <= 9) return launch_fused<9>(a, num_sms, st);
  return launch_fused<17>(a, num_sms, st);  // l > 544: chunked two-pass projection
}

}  // namespace

size_t cgs2_work_bytes(int64_t l, int64_t n, int64_t k, int num_sms) {
  const int64_t G = (int64_t)num_sms * 8;
  size_t b = 0;
  auto add = [&](size_t x) { b += (x + 255) / 256 * 256; };
  add(sizeof(double2) * (size_t)l * (size_t)n);          // W
  add(sizeof(double2) * (size_t)l * (size_t)k);          // Q
  add(sizeof(double2) * (size_t)k * (size_t)l);          // Qh
  add(sizeof(double) * (size_t)rsum_ld(k) * (size_t)l);  // Re Qh + Im Qh (3M GEMM)
  add(sizeof(double2) * (size_t)k * (size_t)n);          // R = Qh Y
  add(sizeof(double2) * (size_t)l);                      // qbuf
  add(sizeof(double2) * (size_t)k);                      // coef
  add(sizeof(Top2) * (size_t)G);                         // per-CTA candidates
  add(sizeof(CgsState));
  add((size_t)n);                                        // chosen flags
  return b;
}

cudaError_t cgs2(double2* Y, int64_t ldy, int64_t l, int64_t n, int64_t k, double tol_rel,
                 const QrcpOut& out, void* work, int num_sms, cudaStream_t stream, int* launches,
                 unsigned long long* trace) {
  if (l > 2048 || k > l || k > n) return cudaErrorInvalidValue;
  char* p = (char*)work;
  auto take = [&](size_t x) {
    char* r = p;
    p += (x + 255) / 256 * 256;
    return (void*)r;
  };
  const int64_t G0 = (int64_t)num_sms * 8;
  double2* W = (double2*)take(sizeof(double2) * (size_t)l * (size_t)n);
  double2* Q = (double2*)take(sizeof(double2) * (size_t)l * (size_t)k);
  double2* Qh = (double2*)take(sizeof(double2) * (size_t)k * (size_t)l);
  double* Qhs = (double*)take(sizeof(double) * (size_t)rsum_ld(k) * (size_t)l);
  double2* R = (double2*)take(sizeof(double2) * (size_t)k * (size_t)n);
  double2* qbuf = (double2*)take(sizeof(double2) * (size_t)l);
  double2* coef = (double2*)take(sizeof(double2) * (size_t)k);
  Top2* cand = (Top2*)take(sizeof(Top2) * (size_t)G0);
  CgsState* st = (CgsState*)take(sizeof(CgsState));
  unsigned char* chosen = (unsigned char*)take((size_t)n);
  cudaError_t e;
  if ((e = cudaMemsetAsync(st, 0, sizeof(CgsState), stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(chosen, 0, (size_t)n, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(out.info, 0, 2 * sizeof(int), stream)) != cudaSuccess) return e;
  if ((e = cudaMemcpy2DAsync(W, sizeof(double2) * l, Y, sizeof(double2) * ldy, sizeof(double2) * l,
                             n, cudaMemcpyDeviceToDevice, stream)) != cudaSuccess)
    return e;
  const unsigned G = (unsigned)std::min<int64_t>(G0, (n + 7) / 8);
  const size_t sm_q = sizeof(double2) * (size_t)l;
  const size_t sm_c = sizeof(double2) * (size_t)k;
  if (sm_q > 48 * 1024 && (e = ensure_dyn_smem((const void*)k_cgs_project, sm_q)) != cudaSuccess)
    return e;
  if (sm_c > 48 * 1024 && (e = ensure_dyn_smem((const void*)k_cgs_update, sm_c)) != cudaSuccess)
    return e;
  int nl = 0;
  const char* ev = select_env("RID_CGS2_FUSED");  // 0: the multi-launch path (tests, measurements)
  bool fused = !(ev && ev[0] == '0');
  if (fused) {
    const char* eo = experiment_env("RID_CGS2_OPT");
    const int opt = eo ? atoi(eo) : 1;
    Cgs2Args a{W, l, n, k, Q, Qh, qbuf, coef, cand, chosen, &st->count, tol_rel, out, opt, trace};
    e = cgs2_fused(a, num_sms, stream);
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      fused = false;
    } else if (e != cudaSuccess) {
      return e;
    } else {
      nl += 1;
    }
  }
  if (!fused) {
  k_cgs_project<<<G, kProjThreads, sm_q, stream>>>(W, l, l, n, qbuf, Q, l, Qh, k, 0, k, tol_rel,
                                                   chosen, st, cand, out.J, out.resid, out.margin,
                                                   out.info);
  ++nl;
  const unsigned gu = (unsigned)((l + 31) / 32);
  for (int64_t j = 0; j < k; ++j) {
    if (j == 0) {
      k_cgs_update<<<gu, 32 * kUpdWarps, 0, stream>>>(Q, l, l, 0, W, l, qbuf, 0, st, coef);
      ++nl;
    } else {
      const unsigned gc = (unsigned)((j + 7) / 8);
      for (int pass = 0; pass < 2; ++pass) {
        k_cgs_coef<<<gc, 256, 0, stream>>>(Q, l, l, j, W, l, qbuf, pass, st, coef);
        k_cgs_update<<<gu, 32 * kUpdWarps, sizeof(double2) * j, stream>>>(Q, l, l, j, W, l, qbuf,
                                                                          pass, st, coef);
        nl += 2;
      }
    }
    k_cgs_project<<<j + 1 < k ? G : 1u, kProjThreads, sm_q, stream>>>(
        W, l, l, n, qbuf, Q, l, Qh, k, j + 1, k, tol_rel, chosen, st, cand, out.J, out.resid,
        out.margin, out.info);
    ++nl;
  }
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // R = Q^H Y on the tensor pipe (a rank failure leaves Q partly unwritten: R is then unused)
  if (sketch_mults() == 3) {
    if ((e = rsum_fill(Qh, k, l, k, Qhs, rsum_ld(k), stream)) != cudaSuccess) return e;
    if ((e = zgemm3m(Qh, k, Qhs, rsum_ld(k), Y, ldy, R, k, k, n, l, stream, 1, nullptr)) !=
        cudaSuccess)
      return e;
    nl += 2;
  } else {
    if ((e = zgemm_ordered(Qh, k, Y, ldy, R, k, k, n, l, 0, 0.0, 0, 0, stream)) != cudaSuccess)
      return e;
    nl += 1;
  }
  k_cgs_r11<<<(unsigned)k, 128, 0, stream>>>(R, k, out.J, k, out.R11, out.beta);
  ++nl;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // the R rows in place of the sketch's first k rows: the contract of the Householder kernels
  // (Y[0:k, c] = R[:, c]) that the solve and rid_qrcp read
  if ((e = cudaMemcpy2DAsync(Y, sizeof(double2) * ldy, R, sizeof(double2) * k, sizeof(double2) * k,
                             n, cudaMemcpyDeviceToDevice, stream)) != cudaSuccess)
    return e;
  if (launches) *launches += nl;
  return cudaSuccess;
}

}  // namespace rid
