// rid_device.cuh — device-side building blocks of the B200 randomized-ID path.
//
// Philox4x32-10 and the RID normal transform, written from the text of docs/RNG.md (§1–§4) with
// explicit IEEE intrinsics (__fma_rn, __dmul_rn, __dadd_rn, __ddiv_rn, __dsqrt_rn) so nvcc can
// neither contract nor reassociate: the result is bit-identical to any other implementation of
// that text (tests/test_gpu_parity.py::test_normal_fill_bitexact checks it against the CPU
// oracle). No code is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rid {

// ---------------------------------------------------------------- Philox4x32-10 (RNG.md §1) --
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;  // the bump after round 10 is dead and removed by the compiler
    k1 += 0xBB67AE85u;
  }
  return c;
}

// ---------------------------------------------------------------- uniforms (RNG.md §3) --------
__device__ __forceinline__ double u01_from(uint32_t lo, uint32_t hi) {
  const unsigned long long w = ((unsigned long long)hi << 32) | lo;
  const double v = __ull2double_rn(w >> 12);  // < 2^52: exact
  return __dmul_rn(__dadd_rn(v, 0.5), 0x1p-52);
}

// ---------------------------------------------------------------- ln u (RNG.md §4.1) ----------
constexpr double kLnC1 = 1.0 / 3.0, kLnC2 = 1.0 / 5.0, kLnC3 = 1.0 / 7.0, kLnC4 = 1.0 / 9.0,
                 kLnC5 = 1.0 / 11.0, kLnC6 = 1.0 / 13.0, kLnC7 = 1.0 / 15.0, kLnC8 = 1.0 / 17.0,
                 kLnC9 = 1.0 / 19.0;

__device__ __forceinline__ double rid_ln(double u) {
  const long long bits = __double_as_longlong(u);
  int e = (int)((bits >> 52) & 0x7FF) - 1023;  // u is normal: u >= 2^-53
  double f = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  if (f > 0x1.6a09e667f3bcdp+0) {
    f = __dmul_rn(f, 0.5);
    e += 1;
  }
  const double s = __ddiv_rn(__dsub_rn(f, 1.0), __dadd_rn(f, 1.0));
  const double z = __dmul_rn(s, s);
  double P = kLnC9;
  P = __fma_rn(P, z, kLnC8);
  P = __fma_rn(P, z, kLnC7);
  P = __fma_rn(P, z, kLnC6);
  P = __fma_rn(P, z, kLnC5);
  P = __fma_rn(P, z, kLnC4);
  P = __fma_rn(P, z, kLnC3);
  P = __fma_rn(P, z, kLnC2);
  P = __fma_rn(P, z, kLnC1);
  const double q = __dmul_rn(z, P);
  const double s2 = __dadd_rn(s, s);
  const double lnf = __fma_rn(s2, q, s2);
  const double de = (double)e;  // exact
  return __dadd_rn(__dmul_rn(de, 0x1.62e42fee00000p-1), __fma_rn(de, 0x1.a39ef35793c76p-33, lnf));
}

// ---------------------------------------------------------------- cos/sin 2πu (RNG.md §4.3) ---
constexpr double kS1 = -1.0 / 6.0, kS2 = 1.0 / 120.0, kS3 = -1.0 / 5040.0, kS4 = 1.0 / 362880.0,
                 kS5 = -1.0 / 39916800.0, kS6 = 1.0 / 6227020800.0, kS7 = -1.0 / 1307674368000.0;
constexpr double kC1 = -1.0 / 2.0, kC2 = 1.0 / 24.0, kC3 = -1.0 / 720.0, kC4 = 1.0 / 40320.0,
                 kC5 = -1.0 / 3628800.0, kC6 = 1.0 / 479001600.0, kC7 = -1.0 / 87178291200.0,
                 kC8 = 1.0 / 20922789888000.0;

__device__ __forceinline__ double2 rid_cossin2pi(double u) {
  const double t = __dmul_rn(4.0, u);
  const double q = rint(t);  // round half to even
  const double r = __dsub_rn(t, q);
  const double x = __dmul_rn(r, 0x1.921fb54442d18p+0);
  const double x2 = __dmul_rn(x, x);
  double Ps = kS7;
  Ps = __fma_rn(Ps, x2, kS6);
  Ps = __fma_rn(Ps, x2, kS5);
  Ps = __fma_rn(Ps, x2, kS4);
  Ps = __fma_rn(Ps, x2, kS3);
  Ps = __fma_rn(Ps, x2, kS2);
  Ps = __fma_rn(Ps, x2, kS1);
  const double sinx = __fma_rn(__dmul_rn(x, x2), Ps, x);
  double Pc = kC8;
  Pc = __fma_rn(Pc, x2, kC7);
  Pc = __fma_rn(Pc, x2, kC6);
  Pc = __fma_rn(Pc, x2, kC5);
  Pc = __fma_rn(Pc, x2, kC4);
  Pc = __fma_rn(Pc, x2, kC3);
  Pc = __fma_rn(Pc, x2, kC2);
  Pc = __fma_rn(Pc, x2, kC1);
  const double cosx = __fma_rn(x2, Pc, 1.0);
  switch (((int)q) & 3) {
    case 0: return make_double2(cosx, sinx);
    case 1: return make_double2(-sinx, cosx);
    case 2: return make_double2(-cosx, -sinx);
    default: return make_double2(sinx, -cosx);
  }
}

// ---------------------------------------------------------------- N(seed, s, i, j) (RNG.md §4) -
__device__ __forceinline__ double2 rid_normal(uint64_t seed, uint32_t s, uint32_t i, uint32_t j) {
  const uint4 x = philox4x32_10(make_uint4(i, j, s, 0u), (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u1 = u01_from(x.x, x.y);
  const double u2 = u01_from(x.z, x.w);
  const double rho = __dsqrt_rn(-rid_ln(u1));
  const double2 cs = rid_cossin2pi(u2);
  return make_double2(__dmul_rn(rho, cs.x), __dmul_rn(rho, cs.y));
}

// ---------------------------------------------------------------- DMMA (FP64 tensor pipe) ------
// mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4. Measured on B200 (profiles/r01_box_facts_*.txt):
// D = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0, C)))) per element, i.e. the K-ascending
// fused chain, bit for bit. Fragment: lane = 4g + t; a = A[g][t] (8x4 row-major),
// b = B[t][g] (4x8), {c0, c1} = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// The same instruction without `volatile`: the compiler may schedule it against the fragment
// loads and adds (each accumulator's chain order is fixed by its data dependence, so the results
// are unchanged).
__device__ __forceinline__ void dmma8x8x4_nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- cp.async helpers -------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int src_bytes = pred ? 16 : 0;  // 0 -> zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------- error-free transformations --
// TwoSum / TwoProd (fma) and a "Dot2" accumulator (Ogita, Rump & Oishi 2005): value = s + c.
struct dd {
  double s, c;
};
__device__ __forceinline__ void dd_add_prod(dd& a, double x, double y) {
  const double p = __dmul_rn(x, y);
  const double pe = __fma_rn(x, y, -p);
  const double s = __dadd_rn(a.s, p);
  const double bv = __dsub_rn(s, a.s);
  const double se = __dadd_rn(__dsub_rn(a.s, __dsub_rn(s, bv)), __dsub_rn(p, bv));
  a.s = s;
  a.c = __dadd_rn(a.c, __dadd_rn(pe, se));
}
__device__ __forceinline__ void dd_add(dd& a, double x) {
  const double s = __dadd_rn(a.s, x);
  const double bv = __dsub_rn(s, a.s);
  const double se = __dadd_rn(__dsub_rn(a.s, __dsub_rn(s, bv)), __dsub_rn(x, bv));
  a.s = s;
  a.c = __dadd_rn(a.c, se);
}
// merge b into a (both Dot2 accumulators)
__device__ __forceinline__ void dd_merge(dd& a, const dd& b) {
  dd_add(a, b.s);
  a.c = __dadd_rn(a.c, b.c);
}
__device__ __forceinline__ double dd_val(const dd& a) { return __dadd_rn(a.s, a.c); }

}  // namespace rid
