// k_crt.cu — the sketch Y = R · A (north_star; §3.1: "Y = R A") on the fifth-generation
// tensor cores (tcgen05, int8 kind) as an EXACT modular integer product (R33):
//
//   1. scale: f_j = b − E_j per column j of A (max |Re|, |Im| of the column < 2^E_j) and e_i = b − E_i
//      per row i of R, so that the integers a' = rint(2^f_j A), r' = rint(2^e_i R) (real and
//      imaginary parts) satisfy |a'|, |r'| <= 2^b;
//   2. residues: for each of T pairwise-coprime odd moduli p_t <= 253, the int8 residues of a' and r'
//      (|residue| <= 127), laid out as the two K-major operands of ONE real product with K' = 2m:
//        Re Y' = [Re r' | −Im r'] · [Re a'; Im a'],   Im Y' = [Im r' | Re r'] · [Re a'; Im a'];
//   3. T products on tcgen05.mma.kind::i8 (int32 accumulators in TMEM, exact: 2m·127² < 2^31 per K
//      slice), each reduced mod p_t in the epilogue;
//   4. the Chinese remainder theorem (Garner's mixed radix, exact 128-bit integers) recovers Y'
//      exactly from its T residues (M = Π p_t > 2 · 4m · 2^2b), and Y = 2^−(e_i+f_j) Y' in fp64.
// Y' is the exact product of the rounded operands: the only errors are the roundings of R and A to
// b bits relative to their row / column maxima (T = 15: b = 50 for m <= 32768, 49 up to 2^17) and
// the final rounding to fp64 — no accumulation error, no Gauss/Strassen cancellation: Y is more
// accurate than an fp64 GEMM's (measured against the oracle in tests/test_gpu_crt.py).
//
// The GEMM kernel (k_imma): persistent, one CTA per SM, 6 warps — warp 0 issues the TMA boxes
// (SWIZZLE_128B, 3D maps over the moduli), warp 1 allocates TMEM and one elected thread issues
// tcgen05.mma, warps 2–5 drain the accumulators (tcgen05.ld) and reduce them mod p_t. The tile is
// 128 columns of A (TMEM lanes) × nc rows of R (TMEM columns, Re at column 0, Im at column 256).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include <cooperative_groups.h>

#include "rid_internal.h"
#include "rid_tma.cuh"

namespace rid {

namespace {

// The moduli: odd, pairwise coprime, <= 253 (so a residue from a quotient that may be off by one
// near a half-integer stays within ±127: crt_res_byte64), descending.
constexpr int kCrtMaxT = 16;
constexpr int kModuli[kCrtMaxT] = {253, 251, 249, 247, 245, 241, 239, 233,
                                   229, 227, 223, 211, 199, 197, 193, 191};

struct CrtConst {
  int T;
  int p[kCrtMaxT];
  float pf[kCrtMaxT], invpf[kCrtMaxT];
  float c16[kCrtMaxT], c32[kCrtMaxT];   // 2^16, 2^32 mod p, symmetric representatives
  double invpd[kCrtMaxT];
  uint32_t magic[kCrtMaxT];             // ceil(2^32 / p): floor(x / p) = umulhi(x, magic), x < 2^21
  uint32_t W[kCrtMaxT][kCrtMaxT];       // W[s][t] = (p_0 ... p_{s-1}) mod p_t
  uint32_t invP[kCrtMaxT];              // (p_0 ... p_{t-1})^{-1} mod p_t
  unsigned long long Mlo, Mhi;          // M = p_0 ... p_{T-1} (< 2^128)
  unsigned long long Hlo, Hhi;          // (M − 1) / 2
};
__constant__ CrtConst c_crt;

__device__ __forceinline__ uint32_t mod_small(uint32_t x, int t) {  // x < 2^21
  const uint32_t q = __umulhi(x, c_crt.magic[t]);
  return x - q * (uint32_t)c_crt.p[t];
}

// ------------------------------------------------------------------ scales --------------------
// rowmax[i] (zeroed by the launcher) = max_k max(|Re R(i, k)|, |Im R(i, k)|); R column-major
__global__ void k_crt_rowmax(const double2* __restrict__ R, int64_t ldr, int64_t l, int64_t m,
                             int64_t kpart, unsigned long long* __restrict__ rowmax) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= l) return;
  const int64_t k0 = blockIdx.y * kpart, k1 = min(m, k0 + kpart);
  double v = 0.0;
  for (int64_t k = k0; k < k1; ++k) {
    const double2 z = R[i + k * ldr];
    v = fmax(v, fmax(fabs(z.x), fabs(z.y)));
  }
  atomicMax(rowmax + i, (unsigned long long)__double_as_longlong(v));  // v >= 0: bits order
}

// the exponent shift s with |x| * 2^s <= 2^b for |x| <= vmax (0 for an all-zero line)
__device__ __forceinline__ int crt_shift(double vmax, int b) {
  if (!(vmax > 0.0)) return 0;
  int E;
  frexp(vmax, &E);  // vmax = f 2^E, f in [0.5, 1): vmax < 2^E
  return b - E;
}

// ------------------------------------------------------------------ residues ------------------
// 2^s as s1 * s2, each a normal double (s > 1000 only for lines whose maximum is below 2^-954)
struct Scale {
  double s1, s2;
};
__device__ __forceinline__ Scale crt_scale(int s) {
  const int a = s > 1000 ? 1000 : s;
  return Scale{ldexp(1.0, a), ldexp(1.0, s - a)};
}
// The residue of a mod p_t from the FP64 pipe: a is the exact integer rint(x 2^s) as a double
// and a_lo its low 32 bits. q = rint(a / p) is one DFMA against 1.5 2^52 (|a| <= 2^50, |a / p| <
// 2^43; the rounded 1/p moves the product by at most 2^50 2^-53 / p < 2^-10, so q is off by one
// only within 2^-10 of a half-integer and |a − p q| <= 0.501 p <= 127), and the remainder's low
// byte comes from 32-bit integer arithmetic on the low words:
// a − p q = a_lo − p q_lo (mod 2^32). One DFMA + one IMAD per residue (round 2's first version
// split a into three fp32 limbs and spent six FP32 operations per residue: C4 preparation 2.98 vs
// 2.42 ms per 8192-column block).
__device__ __forceinline__ uint32_t crt_res_byte64(double a, uint32_t a_lo, int t) {
  const double qb = __fma_rn(a, c_crt.invpd[t], 6755399441055744.0);  // 1.5 2^52 + q
  return a_lo - (uint32_t)c_crt.p[t] * (uint32_t)__double2loint(qb);
}
// a = rint(x scale) as an exact double, and its low 32 bits (|x scale| <= 2^50 < 2^51)
struct Int46 {
  double a;
  uint32_t lo;
};
__device__ __forceinline__ Int46 crt_int46(double x, double scale) {
  const double z = __fma_rn(x, scale, 6755399441055744.0);  // 1.5 2^52 + rint(x 2^s)
  return Int46{z - 6755399441055744.0, (uint32_t)__double2loint(z)};
}
// the low bytes of four words, packed (three PRMTs)
__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}

// A (m x ncols, lda) -> Ares[t][j][k'] (int8, row pitch Kp): k' < mh: Re a'(k, j); mh <= k' < 2mh:
// Im a'(k' − mh, j); zero for k >= m and k' >= 2 mh.
template <int T, bool TWO_STEP>
__device__ __forceinline__ void crt_prep_quads(const double2* __restrict__ a, int64_t m,
                                               int64_t qa, int64_t qbeg, int64_t qend,
                                               int64_t tstride, const Scale scale,
                                               uint32_t* __restrict__ row) {
  for (int64_t q = qbeg + threadIdx.x; q < qend; q += blockDim.x) {
    if (q >= qa) {  // K' padding
      const int64_t w = 2 * qa + (q - qa);
#pragma unroll
      for (int t = 0; t < T; ++t) __stcs(row + t * tstride + w, 0u);
      continue;
    }
    const int64_t k0 = 4 * q;
    Int46 re[4], im[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double2 z = make_double2(0.0, 0.0);
      if (k0 + u < m) z = __ldcs(a + k0 + u);  // last use of A here: evict first
      if (TWO_STEP) {
        z.x *= scale.s1;
        z.y *= scale.s1;
      }
      re[u] = crt_int46(z.x, TWO_STEP ? scale.s2 : scale.s1);
      im[u] = crt_int46(z.y, TWO_STEP ? scale.s2 : scale.s1);
    }
    uint32_t* pr = row + q;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      __stcs(pr, pack4(crt_res_byte64(re[0].a, re[0].lo, t), crt_res_byte64(re[1].a, re[1].lo, t),
                       crt_res_byte64(re[2].a, re[2].lo, t), crt_res_byte64(re[3].a, re[3].lo, t)));
      __stcs(pr + qa,
             pack4(crt_res_byte64(im[0].a, im[0].lo, t), crt_res_byte64(im[1].a, im[1].lo, t),
                   crt_res_byte64(im[2].a, im[2].lo, t), crt_res_byte64(im[3].a, im[3].lo, t)));
      pr += tstride;
    }
  }
}

// The conversion with the column maximum fused in. Default: one CTA per column at a time,
// persistent over columns — it reads the column once for its maximum and again for the residues
// (mostly from L2 at C4: 148 columns of 512 KB in flight; the residue stores and the second read
// are marked evict-first). Experiment (RID_CRT_PREP_CLUSTER): a cluster of CL CTAs per column, each
// reading 1/CL of it, the partial maxima exchanged through distributed shared memory (one cluster
// barrier) — A read from DRAM exactly once, but measured slower (§5.5). Only the maximum's EXPONENT matters (crt_shift), so the first pass takes the
// integer maximum of the high words of |Re|, |Im| — two integer operations per value — and an
// exponent field 0x7FF (inf / NaN) marks the column bad. T is a compile-time constant so the
// modulus loop unrolls with the constants as instruction operands.
template <int T>
__global__ void __launch_bounds__(1024) k_crt_prepA(const double2* __restrict__ A, int64_t lda,
                                                    int64_t m, int64_t ncols, int64_t mh,
                                                    int64_t Kp, double* __restrict__ colmax,
                                                    int b, uint32_t* __restrict__ Ares) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks(), rk = (int)cl.block_rank();
  __shared__ uint32_t red[32];
  __shared__ uint32_t part[2];  // this CTA's partial maximum, by column parity
  __shared__ double red_d[32];
  __shared__ double part_d[2];
  const int64_t qa = mh / 4, qrow = Kp / 4 - qa;  // quads of K per part, + the K' padding words
  const int64_t tstride = ncols * (Kp / 4);
  const int64_t nclu = gridDim.x / CL, cid = blockIdx.x / CL;
  const int64_t kseg = (m + CL - 1) / CL, qseg = (qrow + CL - 1) / CL;
  int par = 0;
  for (int64_t j = cid; j < ncols; j += nclu, par ^= 1) {
    const double2* a = A + j * lda;
    uint32_t hmax = 0;
    const int64_t kb = rk * kseg, ke = min(m, kb + kseg);
    for (int64_t k = kb + threadIdx.x; k < ke; k += blockDim.x) {
      const double2 z = a[k];
      hmax = max(hmax, max((uint32_t)__double2hiint(z.x) & 0x7FFFFFFFu,
                           (uint32_t)__double2hiint(z.y) & 0x7FFFFFFFu));
    }
    hmax = __reduce_max_sync(0xffffffffu, hmax);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = hmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t v = red[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = max(v, red[w]);
      part[par] = v;
    }
    cl.sync();  // every CTA's part[par] is written (and the previous column's reads are done)
    hmax = 0;
    for (int r = 0; r < CL; ++r) hmax = max(hmax, *cl.map_shared_rank(&part[par], r));
    double vmax = __hiloint2double((int)hmax, 0);  // the maximum's exponent, in a double
    const bool bad = hmax >= 0x7FF00000u;
    if (!bad && hmax < 0x00100000u) {  // subnormal or zero column: the exact maximum (rare)
      double v = 0.0;
      for (int64_t k = kb + threadIdx.x; k < ke; k += blockDim.x) {
        const double2 z = a[k];
        v = fmax(v, fmax(fabs(z.x), fabs(z.y)));
      }
      for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if ((threadIdx.x & 31) == 0) red_d[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x == 0) {
        double w0 = red_d[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) w0 = fmax(w0, red_d[w]);
        part_d[par] = w0;
      }
      cl.sync();
      v = 0.0;
      for (int r = 0; r < CL; ++r) v = fmax(v, *cl.map_shared_rank(&part_d[par], r));
      vmax = v;
    }
    if (threadIdx.x == 0 && rk == 0)
      colmax[j] = bad ? __longlong_as_double(0x7ff8000000000000LL) : vmax;
    const int sh = crt_shift(bad ? 0.0 : vmax, b);
    const Scale scale = crt_scale(sh);
    uint32_t* row = Ares + j * (Kp / 4);
    const int64_t qb = rk * qseg, qe = min(qrow, qb + qseg);
    if (sh > 1000)
      crt_prep_quads<T, true>(a, m, qa, qb, qe, tstride, scale, row);
    else
      crt_prep_quads<T, false>(a, m, qa, qb, qe, tstride, scale, row);
    __syncthreads();  // red / red_d are reused by the next column
  }
  cl.sync();  // no CTA exits while a peer may still read its part[] through DSMEM
}

// R (l x m, column-major, ldr) -> Rres[t][0 | 1][lp][Kp]: the operand rows of Re Y' (plane 0:
// [Re r' | −Im r']) and Im Y' (plane 1: [Im r' | Re r']); rows l..lp−1 and the K' padding zero.
// One block: 16 rows x 128 K, staged through shared memory so both the read (down a column of R)
// and the writes (along a row of the operands) are coalesced.
constexpr int kRT_I = 16, kRT_K = 128;
__global__ void __launch_bounds__(256) k_crt_resR(const double2* __restrict__ R, int64_t ldr,
                                                  int64_t l, int64_t m, int64_t lp, int64_t mh,
                                                  int64_t Kp, const unsigned long long* __restrict__ rowmax,
                                                  int b, uint32_t* __restrict__ Rres) {
  __shared__ double2 tile[kRT_K][kRT_I + 1];
  const int64_t i0 = blockIdx.y * (int64_t)kRT_I, k0 = blockIdx.x * (int64_t)kRT_K;
  const int T = c_crt.T;
  const int64_t tstride = 2 * lp * (Kp / 4), pstride = lp * (Kp / 4);
  if (k0 >= mh) {  // K' padding columns [2 mh, Kp): this block writes them for its rows
    const int64_t w0 = 2 * mh / 4, nw = (Kp - 2 * mh) / 4;
    for (int64_t e = threadIdx.x; e < (int64_t)kRT_I * nw; e += blockDim.x) {
      const int64_t ii = e / nw, w = w0 + e % nw, i = i0 + ii;
      if (i >= lp) continue;
      for (int t = 0; t < T; ++t)
        for (int pl = 0; pl < 2; ++pl) Rres[t * tstride + pl * pstride + i * (Kp / 4) + w] = 0u;
    }
    return;
  }
  for (int e = threadIdx.x; e < kRT_I * kRT_K; e += blockDim.x) {
    const int ii = e % kRT_I, kk = e / kRT_I;
    const int64_t i = i0 + ii, k = k0 + kk;
    tile[kk][ii] = (i < l && k < m) ? R[i + k * ldr] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  // thread: row ii, K quad kq
  for (int e = threadIdx.x; e < kRT_I * (kRT_K / 4); e += blockDim.x) {
    const int ii = e / (kRT_K / 4), kq = e % (kRT_K / 4);
    const int64_t i = i0 + ii;
    if (i >= lp) continue;
    const int64_t kw = (k0 + 4 * kq) / 4;  // word index of the quad
    if (4 * kw >= mh) continue;
    const double vmax = i < l ? __longlong_as_double((long long)rowmax[i]) : 0.0;
    const Scale scale = crt_scale(crt_shift(vmax, b));
    const bool two = scale.s2 != 1.0;
    Int46 re[4], im[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double2 z = tile[4 * kq + u][ii];
      if (two) {
        z.x *= scale.s1;
        z.y *= scale.s1;
      }
      re[u] = crt_int46(z.x, two ? scale.s2 : scale.s1);
      im[u] = crt_int46(z.y, two ? scale.s2 : scale.s1);
    }
    uint32_t* base = Rres + i * (Kp / 4);
    for (int t = 0; t < T; ++t) {
      uint32_t br[4], bi[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        br[u] = crt_res_byte64(re[u].a, re[u].lo, t);
        bi[u] = crt_res_byte64(im[u].a, im[u].lo, t);
      }
      const uint32_t wr = pack4(br[0], br[1], br[2], br[3]);
      const uint32_t wi = pack4(bi[0], bi[1], bi[2], bi[3]);
      // −Im r': the negated residues (|r| <= 127, so the negation stays an int8)
      const uint32_t wn = pack4(0u - bi[0], 0u - bi[1], 0u - bi[2], 0u - bi[3]);
      uint32_t* p0 = base + t * tstride;        // plane 0: [Re | −Im]
      uint32_t* p1 = p0 + pstride;              // plane 1: [Im | Re]
      p0[kw] = wr;
      p0[mh / 4 + kw] = wn;
      p1[kw] = wi;
      p1[mh / 4 + kw] = wr;
    }
  }
}

// ------------------------------------------------------------------ tcgen05 GEMM --------------
constexpr int kImmaStagesMax = 8;
constexpr int kImmaThreads = 192;

constexpr int kCrtMaxChunks = 8;  // l <= 2048 rows in tiles of <= 256
struct ImmaArgs {
  int T, kslices, kbps, coltiles, chunks, nc, lp, stages;  // nc: the largest row tile (the box)
  int cn[kCrtMaxChunks], coff[kCrtMaxChunks];              // rows and first row of tile c
  uint32_t cidesc[kCrtMaxChunks];                          // its instruction descriptor
  int64_t n;                // valid A columns
  uint8_t* out;             // [kslices][T][2][n][lp] residues in [0, p)
};

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tma_box3(void* dst, const CUtensorMap* map, int x, int y, int z,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// K-major operand in the canonical swizzled layout of KB-byte rows (KB = 128: SWIZZLE_128B, layout
// type 2; KB = 64: SWIZZLE_64B, type 4): 8-row groups 8 KB bytes apart (stride byte offset),
// leading byte offset 1 (unused when swizzled), version 1 (sm_100)
template <int KB>
__device__ __forceinline__ uint64_t umma_desc_sw(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(8 * KB >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)(KB == 128 ? 2 : 4) << 61);
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// the same with A from tensor memory (kind::i8 .. [d], [a], b_desc): A staged by tcgen05.cp
__device__ __forceinline__ void umma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 128 rows x 32 bytes of a K-major shared-memory operand into tensor memory (8 columns)
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// TS: the A tile of each K step is copied once into tensor memory (tcgen05.cp) and both products
// (Re, Im) read it from there instead of from shared memory: the shared-memory operand traffic per
// K step drops from 2 A + 2 B tiles to 1 A + 2 B (nc <= 192: Re accumulator at TMEM column 0, Im
// at 192, A slots at 384 + 8 (stage 4 / KB·32 + k step))
template <int KB, bool TS>
__global__ void __launch_bounds__(kImmaThreads, 1)
    k_imma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
           const ImmaArgs a) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[kImmaStagesMax], empty[kImmaStagesMax], tfull, tempty;
  __shared__ uint32_t tmem_slot;
  unsigned char* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.stages, nc = a.nc;
  const uint32_t aBytes = 128 * KB, bBytes = (uint32_t)nc * KB;
  const uint32_t stageBytes = aBytes + 2 * bBytes;
  const int nitems = a.T * a.kslices * a.coltiles * a.chunks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 128);
    mbar_init_fence();
    tma_prefetch_map(&mapA);
    tma_prefetch_map(&mapB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(&tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        int r = it;
        const int ch = r % a.chunks; r /= a.chunks;
        const int ct = r % a.coltiles; r /= a.coltiles;
        const int ks = r % a.kslices; r /= a.kslices;
        const int t = r;
        for (int kb = 0; kb < a.kbps; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* st = sm + (size_t)stage * stageBytes;
          mbar_expect_tx(&full[stage], stageBytes);
          const int kx = (ks * a.kbps + kb) * KB;
          tma_box3(st, &mapA, kx, ct * 128, t, &full[stage]);
          tma_box3(st + aBytes, &mapB, kx, a.coff[ch], 2 * t, &full[stage]);
          tma_box3(st + aBytes + bBytes, &mapB, kx, a.coff[ch], 2 * t + 1, &full[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0, iter = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++iter) {
        const uint32_t idesc = a.cidesc[it % a.chunks];
        mbar_wait(&tempty, (iter & 1) ^ 1);  // the epilogue has drained the accumulators
        tc_fence_after();
        for (int kb = 0; kb < a.kbps; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(sm + (size_t)stage * stageBytes);
#pragma unroll
          for (int kk = 0; kk < KB / 32; ++kk) {  // K = 32 bytes per instruction
            const uint64_t da = umma_desc_sw<KB>(sa + 32 * kk);
            const uint64_t dr = umma_desc_sw<KB>(sa + aBytes + 32 * kk);
            const uint64_t di = umma_desc_sw<KB>(sa + aBytes + bBytes + 32 * kk);
            const uint32_t acc = (kb | kk) != 0;
            if (TS) {
              const uint32_t ta = tmem + 384 + 8 * (stage * (KB / 32) + kk);
              tmem_cp_128x256b(ta, da);
              umma_i8_ts(tmem, ta, dr, idesc, acc);
              umma_i8_ts(tmem + 192, ta, di, idesc, acc);
            } else {
              umma_i8(tmem, da, dr, idesc, acc);
              umma_i8(tmem + 256, da, di, idesc, acc);
            }
          }
          umma_commit(&empty[stage]);  // frees the stage when these MMAs have read it
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull);
      }
    }
    __syncwarp();
  } else {  // ---------------- epilogue: warps 2..5 -> TMEM lanes 32 (warp % 4) ...
    const int q = warp & 3;
    const int row = 32 * q + lane;
    uint32_t iter = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++iter) {
      int r = it;
      const int ch = r % a.chunks; r /= a.chunks;
      const int ct = r % a.coltiles; r /= a.coltiles;
      const int ks = r % a.kslices; r /= a.kslices;
      const int t = r;
      mbar_wait(&tfull, iter & 1);
      tc_fence_after();
      const int64_t j = (int64_t)ct * 128 + row;
      const int p = c_crt.p[t];
      const double invp = c_crt.invpd[t];
      for (int ri = 0; ri < 2; ++ri) {
        uint8_t* dst = a.out + ((((int64_t)ks * a.T + t) * 2 + ri) * a.n + j) * a.lp + a.coff[ch];
        for (int c0 = 0; c0 < a.cn[ch]; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + ri * (TS ? 192 : 256) + c0, v);
          uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int x = (int)v[e];
            int rr = x - p * (int)floor((double)x * invp);
            rr += rr < 0 ? p : 0;
            rr -= rr >= p ? p : 0;
            w[e >> 2] |= (uint32_t)rr << (8 * (e & 3));
          }
          if (j < a.n) *reinterpret_cast<uint4*>(dst + c0) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------------ the CTA-pair GEMM --------
// k_imma2: the same products with tcgen05.mma.cta_group::2 — a cluster of two CTAs (one TPC)
// computes a 256-column tile of A against nc rows of R: each CTA holds its own 128 A columns and
// HALF of the R rows (nc / 2 of each plane) in shared memory, the leader (rank 0) issues M = 256
// MMAs that read both CTAs' tiles and write each CTA's own TMEM accumulators, so each SM reads
// only half of the B tile per MMA. Both CTAs' TMA boxes complete on the leader's "full" barrier
// (cp.async.bulk.tensor.cta_group::2); the leader's commits are multicast to both CTAs' "empty"
// and "tfull" barriers; both CTAs' epilogues arrive on the leader's "tempty" barrier.
// N = nc is a multiple of 16: each CTA's half (nc / 2 rows per plane) is whole 8-row SW128 atoms.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
// the shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
__device__ __forceinline__ void tma_box3_2sm(void* dst, const CUtensorMap* map, int x, int y, int z,
                                             uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void umma_i8_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive once on the barrier at this shared-memory offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster)
               : "memory");
}

__global__ void __launch_bounds__(kImmaThreads, 1)
    k_imma2(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
            const ImmaArgs a) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[kImmaStagesMax], empty[kImmaStagesMax], tfull, tempty;
  __shared__ uint32_t tmem_slot;
  unsigned char* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rk = cluster_rank();
  const bool leader = rk == 0;
  const int S = a.stages, nc = a.nc, nh = nc / 2;
  const uint32_t aBytes = 128 * 128, bBytes = (uint32_t)nh * 128;
  const uint32_t stageBytes = aBytes + 2 * bBytes;
  const int coltiles2 = (a.coltiles + 1) / 2;  // 256-column tiles
  const int nitems = a.T * a.kslices * coltiles2 * a.chunks;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 256);  // both CTAs' epilogue threads
    mbar_init_fence();
    tma_prefetch_map(&mapA);
    tma_prefetch_map(&mapB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(&tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  cluster_barrier();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int it = pair; it < nitems; it += npairs) {
        int r = it;
        const int ch = r % a.chunks; r /= a.chunks;
        const int ct2 = r % coltiles2; r /= coltiles2;
        const int ks = r % a.kslices; r /= a.kslices;
        const int t = r;
        for (int kb = 0; kb < a.kbps; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* st = sm + (size_t)stage * stageBytes;
          const uint32_t fb = mapa_u32(smem_u32(&full[stage]), 0);
          if (leader) mbar_expect_tx(&full[stage], 2 * stageBytes);
          const int kx = (ks * a.kbps + kb) * 128;
          tma_box3_2sm(st, &mapA, kx, ct2 * 256 + (int)rk * 128, t, fb);
          const int rb = a.coff[ch] + (int)rk * (a.cn[ch] / 2);  // this CTA's half of the tile
          tma_box3_2sm(st + aBytes, &mapB, kx, rb, 2 * t, fb);
          tma_box3_2sm(st + aBytes + bBytes, &mapB, kx, rb, 2 * t + 1, fb);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (the pair's leader)
      int stage = 0;
      uint32_t phase = 0, iter = 0;
      for (int it = pair; it < nitems; it += npairs, ++iter) {
        const uint32_t idesc = a.cidesc[it % a.chunks];
        mbar_wait(&tempty, (iter & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < a.kbps; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(sm + (size_t)stage * stageBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = umma_desc_sw<128>(sa + 32 * kk);
            const uint64_t dr = umma_desc_sw<128>(sa + aBytes + 32 * kk);
            const uint64_t di = umma_desc_sw<128>(sa + aBytes + bBytes + 32 * kk);
            const uint32_t acc = (kb | kk) != 0;
            umma_i8_2sm(tmem, da, dr, idesc, acc);
            umma_i8_2sm(tmem + 256, da, di, idesc, acc);
          }
          umma_commit_2sm(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2sm(&tfull);
      }
    }
    __syncwarp();
  } else {  // ---------------- epilogue (both CTAs): warps 2..5 -> TMEM lanes 32 (warp % 4) ...
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const uint32_t te = mapa_u32(smem_u32(&tempty), 0);
    uint32_t iter = 0;
    for (int it = pair; it < nitems; it += npairs, ++iter) {
      int r = it;
      const int ch = r % a.chunks; r /= a.chunks;
      const int ct2 = r % coltiles2; r /= coltiles2;
      const int ks = r % a.kslices; r /= a.kslices;
      const int t = r;
      mbar_wait(&tfull, iter & 1);
      tc_fence_after();
      const int64_t j = (int64_t)ct2 * 256 + rk * 128 + row;
      const int p = c_crt.p[t];
      const double invp = c_crt.invpd[t];
      for (int ri = 0; ri < 2; ++ri) {
        uint8_t* dst = a.out + ((((int64_t)ks * a.T + t) * 2 + ri) * a.n + j) * a.lp + a.coff[ch];
        for (int c0 = 0; c0 < a.cn[ch]; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + ri * 256 + c0, v);
          uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int x = (int)v[e];
            int rr = x - p * (int)floor((double)x * invp);
            rr += rr < 0 ? p : 0;
            rr -= rr >= p ? p : 0;
            w[e >> 2] |= (uint32_t)rr << (8 * (e & 3));
          }
          if (j < a.n) *reinterpret_cast<uint4*>(dst + c0) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(te);
    }
  }
  tc_fence_before();
  cluster_barrier();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------------ reconstruction ------------
// One output's value from its T residues x[t] in [0, p_t): Garner's mixed radix
// v_t = (x_t − Σ_{s<t} v_s (p_0..p_{s−1})) (p_0..p_{t−1})^{−1} mod p_t, then
// X = v_0 + p_0 (v_1 + p_1 (v_2 + ...)) exactly (< M < 2^128), the symmetric representative and
// its conversion to fp64 (two roundings at most: |error| <= 2 ulp).
template <int T>
__device__ __forceinline__ double crt_value(uint32_t (&x)[T]) {
#pragma unroll
  for (int t = 1; t < T; ++t) {
    uint32_t acc = 0;
#pragma unroll
    for (int s = 0; s < t; ++s) acc += x[s] * c_crt.W[s][t];
    const uint32_t d = x[t] + (uint32_t)c_crt.p[t] - mod_small(acc, t);
    x[t] = mod_small(mod_small(d, t) * c_crt.invP[t], t);
  }
  unsigned long long lo = x[T - 1];  // the top 7 digits: < 253^7 < 2^64
#pragma unroll
  for (int u = T - 2; u >= T - 7; --u) lo = lo * (unsigned)c_crt.p[u] + x[u];
  unsigned __int128 X = lo;
#pragma unroll
  for (int u = T - 8; u >= 0; --u) X = X * (unsigned)c_crt.p[u] + x[u];
  const unsigned __int128 M = ((unsigned __int128)c_crt.Mhi << 64) | c_crt.Mlo;
  const unsigned __int128 H = ((unsigned __int128)c_crt.Hhi << 64) | c_crt.Hlo;
  const bool neg = X > H;
  const unsigned __int128 mag = neg ? M - X : X;
  const double d = __fma_rn((double)(unsigned long long)(mag >> 64), 18446744073709551616.0,
                            (double)(unsigned long long)mag);
  return neg ? -d : d;
}

// Y(i, j) = 2^−(e_i + f_j) · CRT(residues), i < l, j < ncols. A thread takes four consecutive rows
// of one column: one 32-bit load per (slice, modulus, part) instead of four byte loads.
template <int T>
__global__ void __launch_bounds__(256) k_crt_rec(const uint8_t* __restrict__ res, int kslices,
                                                 int64_t n, int64_t lp, int64_t l, int64_t ncols,
                                                 const unsigned long long* __restrict__ rowmax,
                                                 const double* __restrict__ colmax, int b,
                                                 double2* __restrict__ Y, int64_t ldy) {
  const int64_t l4 = (l + 3) / 4;
  const int64_t total = l4 * ncols;
  const int64_t plane = n * lp / 4;  // words
  const uint32_t* rw = reinterpret_cast<const uint32_t*>(res);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / l4, i0 = 4 * (g - j * l4);
    const double cm = colmax[j];
    const int sj = crt_shift(cm, b);
    const uint32_t* rp = rw + (j * lp + i0) / 4;
    double out[2][4];
#pragma unroll 1
    for (int ri = 0; ri < 2; ++ri) {
      uint32_t w[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        w[t] = __ldcs(rp + (int64_t)(2 * t + ri) * plane);
        if (kslices > 1) {  // add the other slices' residues bytewise, mod p_t
          uint32_t sum[4] = {w[t] & 0xFFu, (w[t] >> 8) & 0xFFu, (w[t] >> 16) & 0xFFu, w[t] >> 24};
          for (int ks = 1; ks < kslices; ++ks) {
            const uint32_t v = __ldcs(rp + (int64_t)((ks * T + t) * 2 + ri) * plane);
            sum[0] += v & 0xFFu;
            sum[1] += (v >> 8) & 0xFFu;
            sum[2] += (v >> 16) & 0xFFu;
            sum[3] += v >> 24;
          }
          w[t] = mod_small(sum[0], t) | mod_small(sum[1], t) << 8 | mod_small(sum[2], t) << 16 |
                 mod_small(sum[3], t) << 24;
        }
      }
#pragma unroll 1
      for (int u = 0; u < 4; ++u) {
        uint32_t x[T];
#pragma unroll
        for (int t = 0; t < T; ++t) x[t] = (w[t] >> (8 * u)) & 0xFFu;
        out[ri][u] = crt_value<T>(x);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u;
      if (i >= l) break;
      const int si = crt_shift(__longlong_as_double((long long)rowmax[i]), b);
      double2 y = make_double2(ldexp(out[0][u], -(si + sj)), ldexp(out[1][u], -(si + sj)));
      if (!(cm <= 1.7976931348623157e308)) y = make_double2(cm, cm);  // inf / NaN: NaN
      Y[j * ldy + i] = y;
    }
  }
}

// ------------------------------------------------------------------ host ---------------------
uint32_t egcd_inv(uint32_t a, uint32_t p) {  // a^{-1} mod p (p prime-power-free coprime)
  int64_t t = 0, nt = 1, r = p, nr = a % p;
  while (nr) {
    const int64_t qq = r / nr;
    int64_t tmp = t - qq * nt; t = nt; nt = tmp;
    tmp = r - qq * nr; r = nr; nr = tmp;
  }
  return (uint32_t)((t % (int64_t)p + p) % p);
}

struct CrtHost {
  CrtConst c;
  double log2M;
};
CrtHost make_const(int T) {
  CrtHost h{};
  CrtConst& c = h.c;
  c.T = T;
  unsigned __int128 M = 1;
  h.log2M = 0;
  for (int t = 0; t < T; ++t) {
    const int p = kModuli[t];
    c.p[t] = p;
    c.pf[t] = (float)p;
    c.invpf[t] = 1.0f / (float)p;
    c.invpd[t] = 1.0 / (double)p;
    auto sym = [&](uint64_t x) { int v = (int)(x % p); return (float)(v > p / 2 ? v - p : v); };
    c.c16[t] = sym(1ull << 16);
    c.c32[t] = sym(1ull << 32);
    c.magic[t] = (uint32_t)(((1ull << 32) + p - 1) / p);
    uint64_t P = 1;  // (p_0 .. p_{t-1}) mod p_t
    for (int s = 0; s < T; ++s) c.W[s][t] = 0;
    for (int s = 0; s < t; ++s) {
      c.W[s][t] = (uint32_t)P;
      P = P * (uint64_t)kModuli[s] % p;
    }
    c.invP[t] = t == 0 ? 1 : egcd_inv((uint32_t)P, p);
    M *= (unsigned)p;
    h.log2M += std::log2((double)p);
  }
  c.Mlo = (unsigned long long)M;
  c.Mhi = (unsigned long long)(M >> 64);
  const unsigned __int128 H = (M - 1) / 2;
  c.Hlo = (unsigned long long)H;
  c.Hhi = (unsigned long long)(H >> 64);
  return h;
}

// the CTA-pair GEMM (k_imma2, cta_group::2): RID_CRT_2SM=1. Measured on one box: ~6% more int8
// ops per second than k_imma at fixed clocks; with 32-row granules its row tiles padded more (C4
// 34.68 vs 34.91 ms, C3 5.37 vs 5.29, C5 116.4 vs 110.7). With 16-row granules (the same tiles as
// k_imma) it draws more power and the step runs under a lower power-capped clock: C4 sketch 36.2-
// 37.1 vs 34.7-34.8 ms (SM 1511-1545 vs 1785-1793 MHz), C5 117.7-119.8 vs 106.1-107.4, C3 equal
// (profiles/r02s16_crt_pair.txt). A tested selection, not the default.
// the pipelined sketch's SM split (experiment RID_CRT_PIPE_SPLIT = SMs for the preparation; 0 =
// the two kernels share the SMs)
int crt_pipe_split(int num_sms) {
  const char* v = experiment_env("RID_CRT_PIPE_SPLIT");
  const int s = v ? atoi(v) : 0;
  return s > 0 && s < num_sms / 2 ? s : 0;
}

bool crt_pair_selected() {
  const char* e = select_env("RID_CRT_2SM");
  return e && atoi(e) != 0;
}

int crt_env_T() {
  const char* e = select_env("RID_CRT_MODULI");
  int T = e ? atoi(e) : 15;
  if (T < 8) T = 8;
  if (T > kCrtMaxT) T = kCrtMaxT;
  return T;
}

}  // namespace

int crt_moduli(int* p, int cap) {
  for (int t = 0; t < kCrtMaxT && t < cap; ++t) p[t] = kModuli[t];
  return kCrtMaxT;
}
double crt_log2M(int T) { return make_const(T).log2M; }

CrtPlan crt_plan(int64_t l, int64_t m) {
  CrtPlan p{};
  p.T = crt_env_T();
  const CrtHost h = make_const(p.T);
  // |Y'| <= 2m 2^2b < M / 2  <=>  2b < log2 M − log2(4m); keep 1/4 bit of margin. b <= 50: the
  // magic-number rint (|a| < 2^51) and the FP64 quotient (crt_res_byte64)
  int b = (int)std::floor((h.log2M - std::log2(4.0 * (double)m) - 0.25) / 2.0);
  p.b = b > 50 ? 50 : b;
  p.mh = (m + 63) / 64 * 64;
  const int64_t K2 = 2 * p.mh;
  const int64_t kmax = (int64_t)(2147483647LL / (127 * 127)) / 128 * 128;  // exact int32 slices
  p.kslices = (int)((K2 + kmax - 1) / kmax);
  p.kbps = (int)(((K2 + 127) / 128 + p.kslices - 1) / p.kslices);
  p.Kp = (int64_t)p.kslices * p.kbps * 128;
  // row tiles: l rounded to the MMA's N granule (16, also for the CTA pair: M = 256 takes any
  // N % 16 == 0 and each CTA's half, N / 2 rows, is whole 8-row swizzle atoms), split into
  // ceil(rows / 256) tiles whose sizes differ by at most one granule (C4: 3 x 176; C5: 144 + 128)
  p.pair = crt_pair_selected();
  const int64_t gran = 16;
  const int64_t units = (l + gran - 1) / gran;
  p.chunks = (int)((units * gran + 255) / 256);
  if (p.chunks > kCrtMaxChunks) p.chunks = kCrtMaxChunks;  // l > 2048: callers use DMMA
  p.nc = 0;
  int64_t off = 0;
  for (int c = 0; c < p.chunks; ++c) {
    const int64_t u = units / p.chunks + (c < units % p.chunks ? 1 : 0);
    p.cn[c] = (int)(u * gran);
    p.coff[c] = (int)off;
    off += u * gran;
    p.nc = std::max(p.nc, p.cn[c]);
  }
  p.lp = off;
  return p;
}

// More K slices than exactness needs when a small sketch's GEMM work items (T x slices x column
// tiles x row tiles) would leave the last wave of num_sms CTAs mostly idle (C3: 15 x 32 items =
// 3.2 waves -> 2 slices, 6.5 waves). The slices' residues are summed mod p, so Y is bitwise the
// same for any slicing; large sketches (>= 8 waves) keep the minimum.
void crt_balance(CrtPlan& p, int64_t ncols, int num_sms) {
  if (num_sms < 1) return;
  const int64_t tiles = (ncols + 127) / 128;
  const int64_t base = (int64_t)p.T * p.chunks * tiles;
  if (base * p.kslices >= 8 * (int64_t)num_sms) return;
  const int64_t kb = (2 * p.mh + 127) / 128;  // 128-byte K blocks of K' = 2 mh
  int best = p.kslices;
  double beff = 0.0;
  for (int ks = p.kslices; ks <= 4; ++ks) {
    if (kb / ks < 16) break;  // keep >= 2048 K per item
    const int64_t items = base * ks;
    const double eff = (double)items / (double)(((items + num_sms - 1) / num_sms) * num_sms);
    if (eff > beff + 0.02) {
      beff = eff;
      best = ks;
    }
  }
  if (best == p.kslices) return;
  p.kslices = best;
  p.kbps = (int)((kb + p.kslices - 1) / p.kslices);
  p.Kp = (int64_t)p.kslices * p.kbps * 128;
}

size_t crt_R_bytes(const CrtPlan& p) {  // Rres + rowmax
  return (size_t)p.T * 2 * p.lp * p.Kp + 8 * (size_t)p.lp + 256;
}
size_t crt_A_bytes(const CrtPlan& p, int64_t ncols) {  // Ares + residues out + colmax
  return (size_t)p.T * ncols * p.Kp + (size_t)p.kslices * p.T * 2 * ncols * p.lp + 8 * (size_t)ncols + 512;
}

namespace {
cudaError_t upload_const(int T, cudaStream_t st) {
  static thread_local int cur_dev = -1, cur_T = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev == cur_dev && T == cur_T) return cudaSuccess;
  const CrtHost h = make_const(T);
  e = cudaMemcpyToSymbolAsync(c_crt, &h.c, sizeof(CrtConst), 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);  // h is a local
  if (e == cudaSuccess) {
    cur_dev = dev;
    cur_T = T;
  }
  return e;
}
}  // namespace

cudaError_t crt_prep_R(const CrtPlan& p, const double2* R, int64_t ldr, int64_t l, int64_t m,
                       void* ws, cudaStream_t st, int* launches) {
  cudaError_t e = upload_const(p.T, st);
  if (e != cudaSuccess) return e;
  uint32_t* Rres = (uint32_t*)ws;
  unsigned long long* rowmax = (unsigned long long*)((char*)ws + (size_t)p.T * 2 * p.lp * p.Kp);
  if ((e = cudaMemsetAsync(rowmax, 0, 8 * (size_t)p.lp, st)) != cudaSuccess) return e;
  const int64_t kpart = std::max<int64_t>(1024, (m + 65534) / 65535);  // grid.y <= 65535
  dim3 g1((unsigned)((l + 127) / 128), (unsigned)((m + kpart - 1) / kpart));
  k_crt_rowmax<<<g1, 128, 0, st>>>(R, ldr, l, m, kpart, rowmax);
  // K blocks cover [0, mh) plus one more block row for the padding [2 mh, Kp)
  const int64_t kblk = (p.mh + kRT_K - 1) / kRT_K + 1;
  dim3 g2((unsigned)kblk, (unsigned)((p.lp + kRT_I - 1) / kRT_I));
  k_crt_resR<<<g2, 256, 0, st>>>(R, ldr, l, m, p.lp, p.mh, p.Kp, rowmax, p.b, Rres);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

namespace {
// bytes of K per pipeline stage: 128 (SWIZZLE_128B, default) or 64 (SWIZZLE_64B: twice the stages
// in flight, measured slower — C4 GEMM 25.2 vs 21.8 ms: the MMAs are bound by shared-memory
// operand bandwidth, not by the depth of the TMA ring)
int crt_kb() {
  const char* e = experiment_env("RID_CRT_KB");
  return e && atoi(e) == 64 ? 64 : 128;
}

// A from tensor memory (k_imma<128, true>) when the row tile allows it (nc <= 192); RID_CRT_TS=0
// keeps both operands in shared memory
// (measured slower: C4 sketch 36.7 vs 34.4 ms, C5 117.8 vs 110.1 — the tensor-memory copy costs
// more than the shared-memory reads it saves; RID_CRT_TS=1 selects it, bitwise the same Y)
bool crt_ts(const CrtPlan& p) {
  if (p.nc > 192) return false;
  const char* e = select_env("RID_CRT_TS");
  return e && atoi(e) != 0;
}

template <int KB, bool TS>
cudaError_t launch_imma(const CrtPlan& p, const uint8_t* Rres, uint8_t* Ares, uint8_t* out,
                        int64_t ncols, int num_sms, cudaStream_t st) {
  cudaError_t e;
  PFN_cuTensorMapEncodeTiled encode;
  if ((e = tensor_map_encoder(&encode)) != cudaSuccess) return e;
  const CUtensorMapSwizzle sw = KB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  CUtensorMap mapA, mapB;
  {
    cuuint64_t gdim[3] = {(cuuint64_t)p.Kp, (cuuint64_t)ncols, (cuuint64_t)p.T};
    cuuint64_t gstr[2] = {(cuuint64_t)p.Kp, (cuuint64_t)p.Kp * ncols};
    cuuint32_t box[3] = {KB, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (encode(&mapA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)Ares, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t gdim[3] = {(cuuint64_t)p.Kp, (cuuint64_t)p.lp, (cuuint64_t)(2 * p.T)};
    cuuint64_t gstr[2] = {(cuuint64_t)p.Kp, (cuuint64_t)p.Kp * p.lp};
    cuuint32_t box[3] = {KB, (cuuint32_t)p.nc, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (encode(&mapB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)Rres, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  ImmaArgs ia{};
  ia.T = p.T;
  ia.kslices = p.kslices;
  ia.kbps = p.kbps * (128 / KB);
  ia.coltiles = (int)((ncols + 127) / 128);
  ia.chunks = p.chunks;
  ia.nc = p.nc;
  ia.lp = (int)p.lp;
  ia.n = ncols;
  ia.out = out;
  // kind::i8: D s32 (bits 4-5 = 2), A and B signed (bits 7-9, 10-12 = 1), both K-major,
  // N >> 3 at bits 17-22, M >> 4 at bits 24-28; one descriptor per row tile (its own N)
  constexpr uint32_t MDIM = 128u >> 4;
  for (int c = 0; c < p.chunks; ++c) {
    ia.cn[c] = p.cn[c];
    ia.coff[c] = p.coff[c];
    ia.cidesc[c] = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.cn[c] >> 3) << 17) | (MDIM << 24);
  }

  const uint32_t stageBytes = 128 * KB + 2 * (uint32_t)p.nc * KB;
  int optin = 0;
  if ((e = optin_smem(&optin)) != cudaSuccess) return e;
  int S = kImmaStagesMax;
  if (const char* v = experiment_env("RID_CRT_STAGES")) S = std::max(2, std::min(kImmaStagesMax, atoi(v)));
  while (S > 2 && (size_t)S * stageBytes + 1024 + 1024 > (size_t)optin) --S;
  if (TS) S = std::min(S, 512 / KB);  // the A slots: 128 TMEM columns
  ia.stages = S;
  const size_t smem = (size_t)S * stageBytes + 1024;
  if ((e = ensure_dyn_smem((const void*)k_imma<KB, TS>, smem)) != cudaSuccess) return e;
  const int nitems = p.T * p.kslices * ia.coltiles * p.chunks;
  const int grid = std::min(nitems, num_sms);
  k_imma<KB, TS><<<grid, kImmaThreads, smem, st>>>(mapA, mapB, ia);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_imma2(const CrtPlan& p, const uint8_t* Rres, uint8_t* Ares, uint8_t* out,
                         int64_t ncols, int num_sms, cudaStream_t st) {
  cudaError_t e;
  PFN_cuTensorMapEncodeTiled encode;
  if ((e = tensor_map_encoder(&encode)) != cudaSuccess) return e;
  CUtensorMap mapA, mapB;
  {
    cuuint64_t gdim[3] = {(cuuint64_t)p.Kp, (cuuint64_t)ncols, (cuuint64_t)p.T};
    cuuint64_t gstr[2] = {(cuuint64_t)p.Kp, (cuuint64_t)p.Kp * ncols};
    cuuint32_t box[3] = {128, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (encode(&mapA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)Ares, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t gdim[3] = {(cuuint64_t)p.Kp, (cuuint64_t)p.lp, (cuuint64_t)(2 * p.T)};
    cuuint64_t gstr[2] = {(cuuint64_t)p.Kp, (cuuint64_t)p.Kp * p.lp};
    cuuint32_t box[3] = {128, (cuuint32_t)(p.nc / 2), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (encode(&mapB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)Rres, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  ImmaArgs ia{};
  ia.T = p.T;
  ia.kslices = p.kslices;
  ia.kbps = p.kbps;
  ia.coltiles = (int)((ncols + 127) / 128);
  ia.chunks = p.chunks;
  ia.nc = p.nc;
  ia.lp = (int)p.lp;
  ia.n = ncols;
  ia.out = out;
  // kind::i8, M = 256 (the pair), N = the row tile's
  constexpr uint32_t MDIM = 256u >> 4;
  for (int c = 0; c < p.chunks; ++c) {
    ia.cn[c] = p.cn[c];
    ia.coff[c] = p.coff[c];
    ia.cidesc[c] = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.cn[c] >> 3) << 17) | (MDIM << 24);
  }

  const uint32_t stageBytes = 128 * 128 + 2 * (uint32_t)(p.nc / 2) * 128;
  int optin = 0;
  if ((e = optin_smem(&optin)) != cudaSuccess) return e;
  int S = kImmaStagesMax;
  while (S > 2 && (size_t)S * stageBytes + 1024 + 1024 > (size_t)optin) --S;
  ia.stages = S;
  const size_t smem = (size_t)S * stageBytes + 1024;
  if ((e = ensure_dyn_smem((const void*)k_imma2, smem)) != cudaSuccess) return e;
  const int nitems = p.T * p.kslices * ((ia.coltiles + 1) / 2) * p.chunks;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kImmaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(2 * std::min(nitems, num_sms / 2)));
  int ncl = 0;
  if ((e = cudaOccupancyMaxActiveClusters(&ncl, (const void*)k_imma2, &cfg)) != cudaSuccess) return e;
  cfg.gridDim = dim3((unsigned)(2 * std::max(1, std::min(std::min(nitems, num_sms / 2), ncl))));
  if ((e = cudaLaunchKernelEx(&cfg, k_imma2, mapA, mapB, ia)) != cudaSuccess) return e;
  return cudaGetLastError();
}

// workspace of one column block (ncols <= nb): A residues, GEMM residues out, colmax
struct CrtBlockWs {
  uint8_t* Ares;
  uint8_t* out;
  double* colmax;
};
static CrtBlockWs carve_block(const CrtPlan& p, void* ws, int64_t nb) {
  CrtBlockWs w;
  w.Ares = (uint8_t*)ws;
  w.out = w.Ares + (size_t)p.T * nb * p.Kp;
  uintptr_t cm = (uintptr_t)(w.out + (size_t)p.kslices * p.T * 2 * nb * p.lp);
  w.colmax = (double*)((cm + 255) & ~(uintptr_t)255);
  return w;
}

// excl > 0: the preparation runs on excl SMs of its own beside a GEMM on the other SMs (the
// pipelined sketch, crt_pipe_split): excl CTAs, each with shared memory the GEMM's CTA cannot sit
// beside, so neither kernel shares an SM with the other
static constexpr size_t kPrepExclSmem = 120 * 1024;
static cudaError_t crt_prep_A(const CrtPlan& p, const CrtBlockWs& w, const double2* A, int64_t lda,
                              int64_t ncols, int64_t m, int num_sms, cudaStream_t st, int excl = 0) {
  // CTAs per cluster (per column): 1 by default (a plain launch). Clusters of 2-8 CTAs read each
  // column from DRAM exactly once (CL = 4: 4.30 vs 6.08 GB per C4 block) but are slower: the
  // kernel is issue-bound, and GPC packing leaves SMs idle (CL = 4: 132 of 148 CTAs resident)
  // a CTA pair per column for the tall matrices (m > 65536: C5's 2 MB columns miss L2 on the
  // second read; measured C5 sketch 104.9 -> 102.8 ms at CL = 2, 105.0 / 106.6 at CL = 4 / 8;
  // C4 unchanged at CL = 2, slower beyond): RID_CRT_PREP_CLUSTER selects
  int CL = m > 65536 ? 2 : 1;
  if (const char* v = select_env("RID_CRT_PREP_CLUSTER")) CL = std::max(1, std::min(8, atoi(v)));
  int thr = 1024;
  if (const char* v = experiment_env("RID_CRT_PREP_THREADS")) thr = std::max(128, std::min(1024, atoi(v)));
  const int64_t nclu = std::max<int64_t>(1, std::min<int64_t>(ncols, num_sms / CL));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclu * CL));
  cfg.blockDim = dim3((unsigned)thr);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  uint32_t* Ares = (uint32_t*)w.Ares;
  cudaError_t e;
  {  // persistent over columns: only as many clusters as can be resident at once (GPC packing)
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;  // (device, CL * 4096 + threads) -> clusters
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    auto key = std::make_pair(dev, CL * 4096 + thr);
    auto it = cache.find(key);
    if (it == cache.end()) {
      int nc = 0;
      if ((e = cudaOccupancyMaxActiveClusters(&nc, (const void*)k_crt_prepA<14>, &cfg)) != cudaSuccess)
        return e;
      it = cache.emplace(key, std::max(1, nc)).first;
    }
    const int64_t fit = std::min<int64_t>(nclu, it->second);
    cfg.gridDim = dim3((unsigned)(fit * CL));
  }
  if (excl > 0) {
    cfg.gridDim = dim3((unsigned)(std::max(1, excl / CL) * CL));
    cfg.dynamicSmemBytes = kPrepExclSmem;
  }
  if (CL == 1) cfg.numAttrs = 0;  // a plain launch: each CTA is its own (implicit) cluster
  switch (p.T) {
#define RID_CRT_PREP(TT)                                                                           \
  case TT:                                                                                         \
    if (excl > 0 && (e = ensure_dyn_smem((const void*)k_crt_prepA<TT>, kPrepExclSmem)) != cudaSuccess) \
      return e;                                                                                    \
    e = cudaLaunchKernelEx(&cfg, k_crt_prepA<TT>, A, lda, m, ncols, p.mh, p.Kp, w.colmax, p.b,    \
                           Ares);                                                                  \
    break;
    RID_CRT_PREP(8) RID_CRT_PREP(9) RID_CRT_PREP(10) RID_CRT_PREP(11) RID_CRT_PREP(12)
    RID_CRT_PREP(13) RID_CRT_PREP(14) RID_CRT_PREP(15) RID_CRT_PREP(16)
#undef RID_CRT_PREP
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

static cudaError_t crt_rec(const CrtPlan& p, const CrtBlockWs& w, const unsigned long long* rowmax,
                           double2* Y, int64_t ldy, int64_t l, int64_t ncols, int num_sms,
                           cudaStream_t st) {
  const int64_t tot = (l + 3) / 4 * ncols;
  const int64_t rb = std::min<int64_t>((tot + 255) / 256, (int64_t)num_sms * 8);
  switch (p.T) {
#define RID_CRT_REC(TT)                                                                            \
  case TT:                                                                                         \
    k_crt_rec<TT><<<(unsigned)rb, 256, 0, st>>>(w.out, p.kslices, ncols, p.lp, l, ncols, rowmax,  \
                                                w.colmax, p.b, Y, ldy);                            \
    break;
    RID_CRT_REC(8) RID_CRT_REC(9) RID_CRT_REC(10) RID_CRT_REC(11) RID_CRT_REC(12)
    RID_CRT_REC(13) RID_CRT_REC(14) RID_CRT_REC(15) RID_CRT_REC(16)
#undef RID_CRT_REC
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int64_t crt_block_cols(const CrtPlan& p, int64_t ncols, int64_t budget_bytes, int num_sms) {
  const int64_t tiles = (ncols + 127) / 128;
  const int64_t maxt = std::max<int64_t>(1, budget_bytes / (int64_t)crt_A_bytes(p, 128));
  if (tiles <= maxt) return tiles * 128;
  // blocks whose GEMM work items (ipc per column tile) fill whole waves of num_sms CTAs, when
  // such a block fits the budget (C4: 148 tiles = 45 waves; C5: 37 tiles = 15 waves), the rest of
  // the columns in a last block
  const int64_t ipc = (int64_t)p.T * p.kslices * p.chunks;
  int64_t g = ipc, h = num_sms > 0 ? num_sms : 1;
  while (h) { const int64_t r = g % h; g = h; h = r; }
  const int64_t unit = (num_sms > 0 ? num_sms : 1) / g;
  if (unit <= maxt) return maxt / unit * unit * 128;
  // otherwise as few blocks as the budget allows, the tiles spread evenly over them
  const int64_t nblk = (tiles + maxt - 1) / maxt;
  return (tiles + nblk - 1) / nblk * 128;
}

cudaError_t crt_sketch(const CrtPlan& p, const void* wsR, const double2* A, int64_t lda, double2* Y,
                       int64_t ldy, int64_t l, int64_t ncols, int64_t m, void* const ws[2],
                       int64_t nb, int num_sms, cudaStream_t st, const CrtPipe* pipe,
                       const CrtTiming* tim, int* launches) {
  if (ncols <= 0) return cudaSuccess;
  cudaError_t e = upload_const(p.T, st);
  if (e != cudaSuccess) return e;
  const uint8_t* Rres = (const uint8_t*)wsR;
  const unsigned long long* rowmax =
      (const unsigned long long*)((const char*)wsR + (size_t)p.T * 2 * p.lp * p.Kp);
  const int KB = crt_kb();
  int gi = 0;  // GEMM launches so far (timing events 2 gi, 2 gi + 1 around launch gi)
  auto rec = [&](cudaEvent_t ev) {
    return tim->external ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                         : cudaEventRecord(ev, st);
  };
  // the split pipeline: the preparation on `split` SMs of its own, the GEMM on the others
  const int split = pipe ? crt_pipe_split(num_sms) : 0;
  auto gemm = [&](const CrtBlockWs& w, int64_t nc) {
    cudaError_t r;
    const int num_sms_g = num_sms - split;
    const bool timed = tim && 2 * gi + 1 < tim->nev;
    if (timed && (r = rec(tim->ev[2 * gi])) != cudaSuccess) return r;
    const bool ts = crt_ts(p);
    r = p.pair ? launch_imma2(p, Rres, w.Ares, w.out, nc, num_sms_g, st)
               : KB == 128 ? (ts ? launch_imma<128, true>(p, Rres, w.Ares, w.out, nc, num_sms_g, st)
                        : launch_imma<128, false>(p, Rres, w.Ares, w.out, nc, num_sms_g, st))
                  : launch_imma<64, false>(p, Rres, w.Ares, w.out, nc, num_sms_g, st);
    if (r == cudaSuccess && timed) r = rec(tim->ev[2 * gi + 1]);
    ++gi;
    if (tim) tim->used = std::min(gi, tim->nev / 2);
    return r;
  };
  // column blocks: the first a quarter of the others (its preparation is the exposed prologue)
  std::vector<std::pair<int64_t, int64_t>> blk;  // (col0, cols)
  {
    const int64_t first = pipe && !split ? std::max<int64_t>(128, nb / 4 / 128 * 128) : nb;
    if (tim) tim->used = 0;
    int64_t j0 = 0;
    while (j0 < ncols) {
      const int64_t c = std::min(blk.empty() ? first : nb, ncols - j0);
      blk.emplace_back(j0, c);
      j0 += c;
    }
  }
  const int nsub = (int)blk.size();
  if (!pipe) {  // one stream: prepare, multiply, reconstruct, block by block
    const CrtBlockWs w = carve_block(p, ws[0], nb);
    for (const auto& bc : blk) {
      if ((e = crt_prep_A(p, w, A + bc.first * lda, lda, bc.second, m, num_sms, st)) != cudaSuccess ||
          (e = gemm(w, bc.second)) != cudaSuccess ||
          (e = crt_rec(p, w, rowmax, Y + bc.first * ldy, ldy, l, bc.second, num_sms, st)) != cudaSuccess)
        return e;
      if (launches) *launches += 3;
    }
    return cudaSuccess;
  }
  // two buffers, two streams: block c's GEMM (main stream, tensor cores) runs beside block c+1's
  // preparation and block c-1's reconstruction (aux stream, ALU and HBM)
  const cudaStream_t ax = pipe->stream;
  const CrtBlockWs w[2] = {carve_block(p, ws[0], nb), carve_block(p, ws[1], nb)};
  if ((e = cudaEventRecord(pipe->fork, st)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(ax, pipe->fork, 0)) != cudaSuccess) return e;
  for (int c = 0; c < 2 && c < nsub; ++c) {
    if ((e = crt_prep_A(p, w[c], A + blk[c].first * lda, lda, blk[c].second, m, num_sms, ax)) != cudaSuccess)
      return e;  // the prologue: the whole machine
    if ((e = cudaEventRecord(pipe->prep[c], ax)) != cudaSuccess) return e;
  }
  for (int c = 0; c < nsub; ++c) {
    const int b = c & 1;
    if ((e = cudaStreamWaitEvent(st, pipe->prep[b], 0)) != cudaSuccess) return e;
    if ((e = gemm(w[b], blk[c].second)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(pipe->gemm[b], st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ax, pipe->gemm[b], 0)) != cudaSuccess) return e;
    if ((e = crt_rec(p, w[b], rowmax, Y + blk[c].first * ldy, ldy, l, blk[c].second, num_sms, ax)) != cudaSuccess)
      return e;
    if (c + 2 < nsub) {
      if ((e = crt_prep_A(p, w[b], A + blk[c + 2].first * lda, lda, blk[c + 2].second, m, num_sms,
                          ax, split)) != cudaSuccess)
        return e;
      if ((e = cudaEventRecord(pipe->prep[b], ax)) != cudaSuccess) return e;
    }
    if (launches) *launches += 3;
  }
  if ((e = cudaEventRecord(pipe->join, ax)) != cudaSuccess) return e;
  return cudaStreamWaitEvent(st, pipe->join, 0);
}

}  // namespace rid
