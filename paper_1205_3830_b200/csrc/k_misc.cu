// k_misc.cu — Philox normal fills (RNG.md §2–§4), identity-block assembly of P (PAPER.md:91-93,
// Eq. 11) and the pivot-column gather B = A[:, J] ("B is found by taking the
// left-most m×k matrix of A" after the permutation of PAPER.md:86).
#include "rid_device.cuh"
#include "rid_internal.h"

namespace rid {

// One thread per entry; consecutive threads walk down a column so the 16-byte stores coalesce.
__global__ void k_normal_fill(uint64_t seed, uint32_t s, int64_t rows, int64_t cols, int64_t row0,
                              int64_t col0, double2* __restrict__ out, int64_t ld) {
  const int64_t total = rows * cols;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q % rows, j = q / rows;
    out[j * ld + i] = rid_normal(seed, s, (uint32_t)(row0 + i), (uint32_t)(col0 + j));
  }
}

cudaError_t normal_fill(uint64_t seed, uint32_t s, int64_t rows, int64_t cols, int64_t row0,
                        int64_t col0, double2* out, int64_t ld, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int64_t total = rows * cols;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;  // grid-stride beyond ~64 waves
  k_normal_fill<<<(unsigned)blocks, 256, 0, st>>>(seed, s, rows, cols, row0, col0, out, ld);
  return cudaGetLastError();
}

__global__ void k_assemble_identity(const int64_t* __restrict__ J, int64_t k, int64_t col0,
                                    int64_t n_loc, double2* __restrict__ P, int64_t ldp) {
  const int64_t t = blockIdx.x;
  const int64_t c = J[t] - col0;
  if (c < 0 || c >= n_loc) return;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x)
    P[c * ldp + i] = make_double2(i == t ? 1.0 : 0.0, 0.0);
}

cudaError_t assemble_identity(const int64_t* J, int64_t k, int64_t col0, int64_t n_loc, double2* P,
                              int64_t ldp, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  k_assemble_identity<<<(unsigned)k, 128, 0, st>>>(J, k, col0, n_loc, P, ldp);
  return cudaGetLastError();
}

// Grid-stride over t (any k). A pivot outside [0, n) sets *bad (read by the caller after its
// synchronisation: RID_EINVAL); its column of B stays as the caller zeroed it.
__global__ void k_gather_columns(const double2* __restrict__ A, int64_t lda, int64_t m,
                                 const int64_t* __restrict__ J, int64_t k, int64_t col0,
                                 int64_t n_loc, int64_t n, double2* __restrict__ B, int64_t ldb,
                                 int* __restrict__ bad) {
  for (int64_t t = blockIdx.y; t < k; t += gridDim.y) {
    const int64_t jt = J[t];
    if (jt < 0 || jt >= n) {
      if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(bad, 1);
      continue;
    }
    const int64_t c = jt - col0;
    if (c < 0 || c >= n_loc) continue;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
      B[t * ldb + i] = A[c * lda + i];
  }
}

cudaError_t gather_columns(const double2* A, int64_t lda, int64_t m, const int64_t* J, int64_t k,
                           int64_t col0, int64_t n_loc, int64_t n, double2* B, int64_t ldb,
                           int* bad, cudaStream_t st) {
  if (k <= 0 || m <= 0) return cudaSuccess;
  int64_t bx = (m + 255) / 256;
  if (bx > 64) bx = 64;
  const unsigned by = (unsigned)(k < 65535 ? k : 65535);
  k_gather_columns<<<dim3((unsigned)bx, by), 256, 0, st>>>(A, lda, m, J, k, col0, n_loc, n, B,
                                                           ldb, bad);
  return cudaGetLastError();
}

// dst = ((src[0] + src[1]) + ...) + src[G-1], elementwise in rank order: the in-process data
// plane's all-reduce (rid_comm_init_local; every rank computes the same bits).
__global__ void k_sum_ranks(RankPtrs src, int G, double* __restrict__ dst, int64_t count) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x) {
    double a = src.p[0][q];
    for (int g = 1; g < G; ++g) a = __dadd_rn(a, src.p[g][q]);
    dst[q] = a;
  }
}

cudaError_t sum_ranks(const RankPtrs& src, int G, double* dst, int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_sum_ranks<<<(unsigned)blocks, 256, 0, st>>>(src, G, dst, count);
  return cudaGetLastError();
}

}  // namespace rid
