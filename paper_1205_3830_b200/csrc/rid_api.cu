// rid_api.cu — the C ABI of include/rid.h: argument checking, workspace, host staging, phase
// timing, NCCL plumbing, and the orchestration of the kernels in k_*.cu. No arithmetic of the
// method runs on the host.
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

extern char** environ;  // POSIX: the RID_* knobs are part of the graph key

#include "../../include/rid.h"
#include "rid_internal.h"

// The data plane of a G-rank communicator: the two collectives the path needs.
// Counts are in doubles; every call is collective (all ranks, same count) and ordered on the
// calling context's stream. Implementations: NCCL (rid_comm_init, one process per GPU) and the
// in-process plane of rid_comm_init_local (G contexts in one process, device copies ordered by
// events; how the tests run the G > 1 path on one GPU).
// This rank's part of a sharded QR (NEXT-3): its sketch block and its QR workspace / outputs.
struct ShardQrPart {
  double2* Y;
  int64_t ldy, l, n_loc, k;
  double tol;
  rid::QrcpOut out;
  rid::QrcpWork w;
};

struct RidComm {
  int rank = 0, nranks = 1;
  virtual ~RidComm() = default;
  // in place: buf holds nranks blocks of `count` doubles, block r is rank r's contribution
  virtual rid_status allgather(rid_ctx* c, double* buf, size_t count) = 0;
  // in place: buf = sum over ranks (bitwise the same on every rank)
  virtual rid_status allreduce_sum(rid_ctx* c, double* buf, size_t count) = 0;
  // the pivoted QR of the G sketch blocks in place (every rank's outputs written, identical);
  // false: this data plane has no sharded QR (the caller all-gathers Y and factors it whole)
  virtual bool has_sharded_qr() const { return false; }
  virtual rid_status qr_sharded(rid_ctx*, const ShardQrPart&, int*) { return RID_EINVAL; }
};

struct rid_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  int num_sms = 148;
  std::string err;
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> ws;
  std::unique_ptr<RidComm> comm;  // null: G = 1
  int rank = 0, nranks = 1;
  cudaEvent_t ev[12] = {};
  // host-A streaming (e2e path): a copy stream and double-buffer events, created on first use
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {}, ev_used[2] = {}, ev_copy0 = nullptr, ev_copy1 = nullptr;
  int sketch_kind = 0;  // RID_SKETCH_GAUSSIAN (north star) or RID_SKETCH_SRFT
  int sketch_engine = 0;  // rid_sketch_engine (RID_ENGINE_AUTO: by the size of the sketch)
  // events around the INT8_CRT engine's GEMM launches (created on first use), and whether the
  // current enqueue is being captured into a graph (events are then recorded as external)
  cudaEvent_t crt_tev[64] = {};
  int crt_timed = 0;    // GEMM launches timed by the last CRT sketch
  int64_t crt_budget = (int64_t)20 << 30;  // workspace budget of the CRT column blocks
  int g_crt_timed = 0;  // ... by the captured graph's
  bool capturing = false;
  int qr_kind = 0;      // RID_QR_HOUSEHOLDER (default) or RID_QR_CGS2
  int qr_dist = 0;      // RID_QR_REPLICATED (default) or RID_QR_SHARDED (NEXT-3)
  // pinned host mirror of the QR's status block (info, beta, resid, margin): one copy, one sync
  void* host_qr = nullptr;
  size_t host_qr_bytes = 0;
  // aux stream for the sketch's K-split tail set (rid::SketchAux), created on first use
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
  // the modular integer sketch's column-block pipeline (k_crt.cu), created on first use
  rid::CrtPipe crt_pipe{};
  // CUDA graph of rid_decompose's device work (repeated calls with identical arguments): the
  // key of the last call seen, the captured executable and its key; ws_epoch counts workspace
  // reallocations (a graph holds workspace pointers)
  unsigned long long ws_epoch = 0;
  std::string g_seen, g_key, g_bad;
  cudaGraphExec_t g_exec = nullptr;
  int g_launches = 0;
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t g_in = nullptr, g_out = nullptr;
};

namespace {
// The engine of the Gaussian sketch of an l x m sketch matrix over n columns (rid_sketch_engine):
// RID_SKETCH_CRT in the environment, else the context's selection, else by size
bool use_crt(const rid_ctx* c, int64_t l, int64_t m, int64_t n) {
  // the engine's row tiles: at most 8 of 256 (rid_decompose's bound); K' = 2m bytes of residues
  // per column addressed by int32 TMA coordinates
  if (l > 2048 || m > ((int64_t)1 << 28)) return false;
  if (const char* e = rid::select_env("RID_SKETCH_CRT")) return atoi(e) != 0;
  if (c->sketch_engine == RID_ENGINE_FP64_DMMA) return false;
  if (c->sketch_engine == RID_ENGINE_INT8_CRT) return true;
  return (double)l * (double)m * (double)n >= 17179869184.0;  // 2^34: C3, C4, C5
}
bool strassen_on(const rid_ctx* c, int64_t l, int64_t m, int64_t n) {
  return !use_crt(c, l, m, n) && rid::strassen_plan(l, m, n, c->num_sms);
}
}  // namespace

namespace {

rid_status fail(rid_ctx* c, rid_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return st;
}

#define RID_CUDA(c, expr)                                                                    \
  do {                                                                                       \
    cudaError_t e__ = (expr);                                                                \
    if (e__ != cudaSuccess)                                                                  \
      return fail((c), e__ == cudaErrorMemoryAllocation ? RID_ENOMEM : RID_ECUDA,            \
                  "%s: %s (%s:%d)", #expr, cudaGetErrorString(e__), __FILE__, __LINE__);     \
  } while (0)

#define RID_NCCL(c, expr)                                                                    \
  do {                                                                                       \
    ncclResult_t r__ = (expr);                                                               \
    if (r__ != ncclSuccess)                                                                  \
      return fail((c), RID_ENCCL, "%s: %s", #expr, ncclGetErrorString(r__));                 \
  } while (0)

#define RID_TRY(expr)                 \
  do {                                \
    rid_status s__ = (expr);          \
    if (s__ != RID_OK) return s__;    \
  } while (0)

rid_status ws_get(rid_ctx* c, const char* name, size_t bytes, void** out) {
  auto& b = c->ws[name];
  if (b.bytes < bytes) {
    ++c->ws_epoch;
    if (b.p) {
      RID_CUDA(c, cudaStreamSynchronize(c->stream));
      RID_CUDA(c, cudaFree(b.p));
      b.p = nullptr;
      b.bytes = 0;
    }
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, RID_ENOMEM, "workspace '%s': cudaMalloc(%zu) failed: %s", name, bytes,
                  cudaGetErrorString(e));
    }
    b.bytes = bytes;
  }
  *out = b.p;
  return RID_OK;
}

// ---- NCCL data plane (one process per GPU) ----------------------------------------------------
struct NcclComm final : RidComm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  rid_status allgather(rid_ctx* c, double* buf, size_t count) override {
    RID_NCCL(c, ncclAllGather(buf + (size_t)rank * count, buf, count, ncclDouble, comm, c->stream));
    return RID_OK;
  }
  rid_status allreduce_sum(rid_ctx* c, double* buf, size_t count) override {
    RID_NCCL(c, ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm, c->stream));
    return RID_OK;
  }
};

// ---- in-process data plane (rid_comm_init_local) -----------------------------------------------
// G contexts of one process and one device. A collective is two host rendezvous of the G calling
// threads (like NCCL, every rank must call it) around stream-ordered device work:
//   1. each rank publishes its buffer and records `ready` on its stream; rendezvous;
//   2. each rank's stream waits for every peer's `ready`, then copies / reduces from the peers'
//      buffers (plain device copies, a rank-ordered sum kernel); records `done`; rendezvous;
//   3. each rank's stream waits for every peer's `done` before anything after the collective can
//      overwrite the buffer the peers read.
// No kernel waits on another: the only cross-rank dependencies are stream waits on events
// recorded before the rendezvous, so the G streams may run in any order on the one GPU.
struct LocalGroup {
  int G = 0;
  int device = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long phase = 0;
  bool broken = false;
  std::vector<double*> buf;
  std::vector<ShardQrPart> qr;  // the sharded QR's per-rank parts
  rid_status qr_status = RID_OK;
  std::string qr_err;
  std::vector<cudaEvent_t> ready, done;
  ~LocalGroup() {
    cudaSetDevice(device);
    for (auto e : ready) cudaEventDestroy(e);
    for (auto e : done) cudaEventDestroy(e);
  }
};

struct LocalComm final : RidComm {
  std::shared_ptr<LocalGroup> g;
  rid_status rendezvous(rid_ctx* c) {
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->broken) return fail(c, RID_ENCCL, "local communicator: a rank failed or timed out");
    const unsigned long long ph = g->phase;
    if (++g->arrived == g->G) {
      g->arrived = 0;
      ++g->phase;
      g->cv.notify_all();
      return RID_OK;
    }
    const bool ok = g->cv.wait_for(lk, std::chrono::seconds(300),
                                   [&] { return g->phase != ph || g->broken; });
    if (!ok || g->broken) {
      g->broken = true;
      g->cv.notify_all();
      return fail(c, RID_ENCCL, "local communicator: rank %d timed out at a collective", rank);
    }
    return RID_OK;
  }
  rid_status publish(rid_ctx* c, double* buf) {
    g->buf[rank] = buf;
    RID_CUDA(c, cudaEventRecord(g->ready[rank], c->stream));
    return rendezvous(c);
  }
  rid_status finish(rid_ctx* c) {
    RID_CUDA(c, cudaEventRecord(g->done[rank], c->stream));
    RID_TRY(rendezvous(c));
    for (int h = 0; h < g->G; ++h)
      if (h != rank) RID_CUDA(c, cudaStreamWaitEvent(c->stream, g->done[h], 0));
    return RID_OK;
  }
  rid_status allgather(rid_ctx* c, double* buf, size_t count) override {
    RID_TRY(publish(c, buf));
    for (int h = 0; h < g->G; ++h) {
      if (h == rank) continue;
      RID_CUDA(c, cudaStreamWaitEvent(c->stream, g->ready[h], 0));
      RID_CUDA(c, cudaMemcpyAsync(buf + (size_t)h * count, g->buf[h] + (size_t)h * count,
                                  count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
    return finish(c);
  }
  rid_status allreduce_sum(rid_ctx* c, double* buf, size_t count);
  bool has_sharded_qr() const override { return g->G <= rid::kQrMaxRanks; }
  rid_status qr_sharded(rid_ctx* c, const ShardQrPart& part, int* launches) override;
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// A matrix argument: device pointer used in place, or a host buffer staged in workspace.
struct MatArg {
  void* dev = nullptr;
  bool host = false;
};

rid_status stage_in(rid_ctx* c, const char* name, const void* user, size_t rows, size_t cols,
                    size_t ld, size_t elem, bool copy, MatArg* out) {
  out->host = !is_device_ptr(user);
  if (!out->host) {
    out->dev = const_cast<void*>(user);
    return RID_OK;
  }
  const size_t bytes = (cols == 0 ? 0 : ((cols - 1) * ld + rows)) * elem;
  RID_TRY(ws_get(c, name, bytes ? bytes : elem, &out->dev));
  if (copy && bytes)
    RID_CUDA(c, cudaMemcpyAsync(out->dev, user, bytes, cudaMemcpyHostToDevice, c->stream));
  return RID_OK;
}

rid_status stage_out(rid_ctx* c, const MatArg& a, void* user, size_t rows, size_t cols, size_t ld,
                     size_t elem) {
  if (!a.host) return RID_OK;
  const size_t bytes = (cols == 0 ? 0 : ((cols - 1) * ld + rows)) * elem;
  if (bytes) RID_CUDA(c, cudaMemcpyAsync(user, a.dev, bytes, cudaMemcpyDeviceToHost, c->stream));
  return RID_OK;
}

rid_status check_ctx(rid_ctx* c) {
  if (!c) return RID_EINVAL;
  c->err.clear();
  RID_CUDA(c, cudaSetDevice(c->device));
  return RID_OK;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

constexpr double kRankTol = 1e-13;   // reading R13
constexpr double kSingTol = 1e-13;
constexpr uint32_t kStreamR = 4, kStreamRRetry = 20;

// T = R11^-1 R12 for the shard's columns (reading R29), on the same complex-product kernel as
// the sketch (Gauss's three products by default, R31), written straight into P_loc.
// With the context's aux stream (created by the sketch) the product goes through sketch_gemm, so
// k = 48 a + r (r = 24/32/40; C3 128, C4 512) runs its last r rows of T on r-row tiles beside the
// 48-row launch (bitwise the same T). Adds its kernel launches to *launches.
rid_status solve_T(rid_ctx* c, const double2* Rinv, int64_t k, const double2* Y, int64_t ldy,
                   double2* P, int64_t ldp, int64_t n_loc, int* launches = nullptr,
                   bool crt = false) {
  int dummy = 0;
  if (!launches) launches = &dummy;
  if (crt && rid::select_env("RID_SOLVE_CRT") && atoi(rid::select_env("RID_SOLVE_CRT")) != 0) {
    // the INT8_CRT engine of the sketch (R33) for T = R11^-1 R12 as well: P = Rinv Y[0:k, :].
    // Measured slower at C4 (2.98 vs 2.05 ms: the k x n CRT reconstruction costs more than the
    // DMMA GEMM it replaces), so a tested selection, not the default.
    const rid::CrtPlan cp = rid::crt_plan(k, k);
    void *pr, *pa;
    RID_TRY(ws_get(c, "Rcrt_solve", rid::crt_R_bytes(cp), &pr));
    RID_CUDA(c, rid::crt_prep_R(cp, Rinv, k, k, k, pr, c->stream, launches));
    const int64_t nb = rid::crt_block_cols(cp, n_loc, (int64_t)2 << 30, c->num_sms);
    RID_TRY(ws_get(c, "Acrt_solve", rid::crt_A_bytes(cp, nb), &pa));
    void* pw[2] = {pa, nullptr};
    RID_CUDA(c, rid::crt_sketch(cp, pr, Y, ldy, P, ldp, k, n_loc, k, pw, nb, c->num_sms, c->stream,
                                nullptr, nullptr, launches));
    return RID_OK;
  }
  if (rid::sketch_mults() == 3) {
    void* ps;
    RID_TRY(ws_get(c, "Rinvs", sizeof(double) * rid::rsum_ld(k) * k, &ps));
    RID_CUDA(c, rid::rsum_fill(Rinv, k, k, k, (double*)ps, rid::rsum_ld(k), c->stream));
    *launches += 1;
    if (c->aux_stream && !rid::select_env("RID_SOLVE_NOAUX")) {
      const rid::SketchAux aux{c->aux_stream, c->aux_fork, c->aux_join};
      RID_CUDA(c, rid::sketch_gemm(Rinv, k, (const double*)ps, Y, ldy, P, ldp, k, n_loc, k,
                                   c->stream, 1, nullptr, 0, n_loc, c->num_sms, launches, &aux));
    } else {
      RID_CUDA(c, rid::zgemm3m(Rinv, k, (const double*)ps, rid::rsum_ld(k), Y, ldy, P, ldp, k,
                               n_loc, k, c->stream, 1, nullptr));
      *launches += 1;
    }
  } else {
    RID_CUDA(c, rid::zgemm_ordered(Rinv, k, Y, ldy, P, ldp, k, n_loc, k, 0, 0.0, 0, 0, c->stream));
    *launches += 1;
  }
  return RID_OK;
}

// Factor the full sketch in workspace "Y" and solve for the local shard columns.
// On entry Yw holds the full l x n sketch (ld = l). Writes J (device ws), P_loc (device).
rid_status qr_check(rid_ctx* c, int64_t k, int* info_host, rid_diag* diag);

// defer = true (rid_decompose): enqueue the QR and the copy of its status block, return without
// synchronising; the caller synchronises once at its end and calls qr_check.
// sharded = true (rid_decompose with RID_QR_SHARDED): Yw is this rank's l x n block (n = n_loc)
// and the QR is the communicator's collective sharded QR (NEXT-3).
rid_status factor_and_solve(rid_ctx* c, double2* Yw, int64_t l, int64_t n, int64_t k, int64_t col0,
                            int64_t n_loc, double2* Pdev, int64_t ldp, int64_t** Jdev_out,
                            int* info_host, rid_diag* diag, bool solve, double** beta_out,
                            bool defer = false, bool sharded = false) {
  void *pJ, *pbeta, *presid, *pmargin, *pinfo, *pwork, *pstat;
  RID_TRY(ws_get(c, "J", sizeof(int64_t) * k, &pJ));
  // the QR's status block, contiguous so the host reads it with one copy: info (2 ints, 16 B),
  // then beta, resid, margin (k doubles each)
  const size_t stat_bytes = 16 + 3 * sizeof(double) * (size_t)k;
  RID_TRY(ws_get(c, "qr_status", stat_bytes, &pstat));
  pinfo = pstat;
  pbeta = (char*)pstat + 16;
  presid = (double*)pbeta + k;
  pmargin = (double*)presid + k;
  const int max_blocks = 4 * c->num_sms;
  RID_TRY(ws_get(c, "qrcp_work", rid::qrcp_work_bytes(n, l, max_blocks), &pwork));
  void* pR11;
  RID_TRY(ws_get(c, "R11", sizeof(double2) * k * k, &pR11));
  rid::QrcpOut o{(int64_t*)pJ, (double*)pbeta, (double*)presid, (double*)pmargin, (int*)pinfo,
                 (double2*)pR11};
  rid::QrcpWork w = rid::qrcp_work_carve(pwork, n, l, max_blocks);
  const char* trace_path = rid::select_env("RID_QRCP_TRACE");  // per-step timing of k_qrcp (tools)
  if (trace_path) {
    void* pt;
    RID_TRY(ws_get(c, "qrcp_trace", sizeof(unsigned long long) * 8 * k, &pt));
    RID_CUDA(c, cudaMemsetAsync(pt, 0, sizeof(unsigned long long) * 8 * k, c->stream));
    w.trace = (unsigned long long*)pt;
  }
  RID_CUDA(c, cudaMemsetAsync(pR11, 0, sizeof(double2) * k * k, c->stream));
  if (sharded) {
    const ShardQrPart part{Yw, l, l, n, k, kRankTol, o, w};
    RID_TRY(c->comm->qr_sharded(c, part, diag ? &diag->launches : nullptr));
  } else if (c->qr_kind == RID_QR_CGS2) {  // the paper's own QR
    void* pc;
    RID_TRY(ws_get(c, "cgs2_work", rid::cgs2_work_bytes(l, n, k, c->num_sms), &pc));
    RID_CUDA(c, rid::cgs2(Yw, l, l, n, k, kRankTol, o, pc, c->num_sms, c->stream,
                          diag ? &diag->launches : nullptr, w.trace));
  } else {
    RID_CUDA(c, rid::qrcp(Yw, l, l, n, k, kRankTol, o, w, c->num_sms, c->stream,
                          diag ? &diag->launches : nullptr));
  }
  if (trace_path) {
    std::vector<unsigned long long> tr(8 * k);
    RID_CUDA(c, cudaMemcpyAsync(tr.data(), w.trace, sizeof(unsigned long long) * 8 * k,
                                cudaMemcpyDeviceToHost, c->stream));
    RID_CUDA(c, cudaStreamSynchronize(c->stream));
    if (FILE* f = fopen(trace_path, "w")) {
      for (int64_t j = 0; j < k; ++j) {
        fprintf(f, "%lld", (long long)j);
        for (int q = 0; q < 8; ++q) fprintf(f, " %llu", tr[8 * j + q]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  // one synchronisation: rank status, R11 diagonal (singularity), diagnostics — the status block
  // in one copy into the context's pinned mirror (pageable copies cost a round trip each)
  if (c->host_qr_bytes < stat_bytes) {
    ++c->ws_epoch;
    if (c->host_qr) cudaFreeHost(c->host_qr);
    c->host_qr = nullptr;
    c->host_qr_bytes = 0;
    RID_CUDA(c, cudaMallocHost(&c->host_qr, stat_bytes));
    c->host_qr_bytes = stat_bytes;
  }
  RID_CUDA(c, cudaMemcpyAsync(c->host_qr, pstat, stat_bytes, cudaMemcpyDeviceToHost, c->stream));
  *Jdev_out = (int64_t*)pJ;
  if (beta_out) *beta_out = (double*)pbeta;
  if (defer) return RID_OK;
  RID_CUDA(c, cudaStreamSynchronize(c->stream));
  RID_TRY(qr_check(c, k, info_host, diag));
  if (!solve) return RID_OK;
  void* pRinv;
  RID_TRY(ws_get(c, "Rinv", sizeof(double2) * k * k, &pRinv));
  RID_CUDA(c, rid::tri_inverse((const double2*)pR11, k, (double2*)pRinv, c->stream));
  RID_TRY(solve_T(c, (const double2*)pRinv, k, Yw + col0 * l, l, Pdev, ldp, n_loc));
  RID_CUDA(c, rid::assemble_identity((const int64_t*)pJ, k, col0, n_loc, Pdev, ldp, c->stream));
  return RID_OK;
}

// Reads the QR's status block from the pinned mirror (after the caller's synchronisation): rank
// status, R11 diagonal (singularity), diagnostics.
rid_status qr_check(rid_ctx* c, int64_t k, int* info_host, rid_diag* diag) {
  const int* hinfo = (const int*)c->host_qr;
  info_host[0] = hinfo[0];
  info_host[1] = hinfo[1];
  const double* hb = (const double*)((const char*)c->host_qr + 16);
  const double* hr = hb + k;
  const double* hm = hr + k;
  if (diag) {
    const int kk = info_host[0] == 0 ? (int)k : info_host[1];
    double mm = INFINITY;
    for (int j = 0; j + 1 < kk; ++j) mm = std::fmin(mm, hm[j]);
    diag->tie_margin_min = mm;
    diag->rank_achieved = info_host[0] == 0 ? (int)k : info_host[1];
    diag->resid_last = kk > 0 ? hr[kk - 1] : 0.0;
  }
  if (info_host[0] != 0) return RID_ERANK;
  double dmax = 0.0;
  for (int64_t t = 0; t < k; ++t) dmax = std::fmax(dmax, std::fabs(hb[t]));
  for (int64_t t = 0; t < k; ++t)
    if (std::fabs(hb[t]) < kSingTol * dmax)
      return fail(c, RID_ESINGULAR, "R11[%lld,%lld] = %g below 1e-13 * %g", (long long)t,
                  (long long)t, hb[t], dmax);
  return RID_OK;
}

// The sketch matrix in the form the planned kernel reads: R (l x m) and Re R + Im R for the 3M
// kernel, or (Strassen plan, k_strassen.cu) R's seven block combinations and their Re + Im planes.
struct SketchR {
  double2* R = nullptr;
  double* Rs = nullptr;
  bool strassen = false;
  double2* Rc = nullptr;
  double* Rsc = nullptr;
  rid::StrassenWs sw{};
  bool crt = false;  // the modular integer sketch on the int8 tensor cores (k_crt.cu)
  rid::CrtPlan cp{};
  void* crtR = nullptr;
};

// R (l x m, stream s) for the sketch of an m x n matrix, in the form of the plan (l, m, n) picks.
// Adds its launches.
rid_status fill_R(rid_ctx* c, uint64_t seed, uint32_t s, int64_t l, int64_t m, int64_t n,
                  SketchR* out, int* launches) {
  void *pR, *pRs = nullptr;
  RID_TRY(ws_get(c, "R", sizeof(double2) * l * m, &pR));
  rid::sketch_key() = rid::SketchKey{seed, s};
  RID_CUDA(c, rid::normal_fill(seed, s, l, m, 0, 0, (double2*)pR, l, c->stream));
  *launches += 1;
  *out = SketchR{};
  out->R = (double2*)pR;
  if (use_crt(c, l, m, n)) {
    out->crt = true;
    out->cp = rid::crt_plan(l, m);
    if (!rid::select_env("RID_CRT_NOBALANCE")) rid::crt_balance(out->cp, n, c->num_sms);
    RID_TRY(ws_get(c, "Rcrt", rid::crt_R_bytes(out->cp), &out->crtR));
    RID_CUDA(c, rid::crt_prep_R(out->cp, (const double2*)pR, l, l, m, out->crtR, c->stream,
                                launches));
  } else if (strassen_on(c, l, m, n)) {
    out->strassen = true;
    out->sw = rid::strassen_ws(l, m, 0);
    void *pc, *ps;
    RID_TRY(ws_get(c, "Rstr", out->sw.rc_bytes, &pc));
    RID_TRY(ws_get(c, "Rsstr", out->sw.rs_bytes, &ps));
    RID_CUDA(c, rid::strassen_rcomb((const double2*)pR, l, m, l, (double2*)pc, out->sw.ldc,
                                    (double*)ps, out->sw.lds, c->stream));
    *launches += 1;
    out->Rc = (double2*)pc;
    out->Rsc = (double*)ps;
  } else if (rid::sketch_mults() == 3) {
    RID_TRY(ws_get(c, "Rs", sizeof(double) * rid::rsum_ld(l) * m, &pRs));
    RID_CUDA(c, rid::rsum_fill((const double2*)pR, l, m, l, (double*)pRs, rid::rsum_ld(l),
                               c->stream));
    *launches += 1;
    out->Rs = (double*)pRs;
  }
  return RID_OK;
}

// The aux stream and its fork/join events (created on first use) unless RID_SKETCH_NOAUX
rid_status sketch_aux(rid_ctx* c, rid::SketchAux* aux, const rid::SketchAux** out) {
  *out = nullptr;
  if (rid::select_env("RID_SKETCH_NOAUX")) return RID_OK;
  if (!c->aux_stream) {
    RID_CUDA(c, cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
    RID_CUDA(c, cudaEventCreateWithFlags(&c->aux_fork, cudaEventDisableTiming));
    RID_CUDA(c, cudaEventCreateWithFlags(&c->aux_join, cudaEventDisableTiming));
  }
  *aux = rid::SketchAux{c->aux_stream, c->aux_fork, c->aux_join};
  *out = aux;
  return RID_OK;
}

// Y[:, 0:ncols] = R A for the columns [col0, col0 + ncols) of the m x n matrix, by the plan of sr
rid_status sketch_block(rid_ctx* c, const SketchR& sr, const double2* A, int64_t lda, double2* Y,
                        int64_t ldy, int64_t l, int64_t ncols, int64_t m, int64_t col0, int64_t n,
                        int S, double2* partial, int* launches, const rid::SketchAux* aux) {
  int dummy = 0;
  if (!launches) launches = &dummy;
  if (sr.crt) {  // column blocks whose residues fit the workspace budget, pipelined on 2 streams
    // the two-stream block pipeline measured slower (the residue kernels beside the GEMM slow it
    // from 6.0 to 8.4 ms per block): an experiment
    const char* pv = rid::experiment_env("RID_CRT_PIPE");
    const bool piped = pv && atoi(pv) != 0;
    // column blocks of at most 20 GiB of residues (C4: 148 + 108 column tiles; C5: 37-tile
    // blocks), and at most half of the memory free beside the workspace already held
    // (queried outside graph capture only; a capture reuses the last eager call's budget)
    int64_t budget = c->crt_budget;
    if (!c->capturing) {
      budget = (int64_t)20 << 30;
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
        const auto it = c->ws.find("Acrt0");
        const int64_t held = it != c->ws.end() ? (int64_t)it->second.bytes : 0;
        budget = std::min(budget, std::max<int64_t>((int64_t)1 << 30, ((int64_t)fr + held) / 2));
      }
      c->crt_budget = budget;
    }
    int64_t nb = rid::crt_block_cols(sr.cp, ncols, budget, c->num_sms);
    if (const char* v = rid::experiment_env("RID_CRT_PIPE_NB"))  // pipelined blocks (columns)
      if (piped && atoll(v) >= 128) nb = std::min<int64_t>(nb, atoll(v) / 128 * 128);
    void* pw[2] = {nullptr, nullptr};
    RID_TRY(ws_get(c, "Acrt0", rid::crt_A_bytes(sr.cp, nb), &pw[0]));
    if (piped) {
      RID_TRY(ws_get(c, "Acrt1", rid::crt_A_bytes(sr.cp, nb), &pw[1]));
      if (!c->crt_pipe.stream) {
        RID_CUDA(c, cudaStreamCreateWithFlags(&c->crt_pipe.stream, cudaStreamNonBlocking));
        cudaEvent_t* evs[6] = {&c->crt_pipe.fork, &c->crt_pipe.join, &c->crt_pipe.prep[0],
                               &c->crt_pipe.prep[1], &c->crt_pipe.gemm[0], &c->crt_pipe.gemm[1]};
        for (auto* e : evs) RID_CUDA(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      }
    }
    if (!c->crt_tev[0])
      for (auto& e : c->crt_tev) RID_CUDA(c, cudaEventCreate(&e));
    const rid::CrtTiming tim{c->crt_tev, 64, c->capturing, 0};
    c->crt_timed = 0;
    RID_CUDA(c, rid::crt_sketch(sr.cp, sr.crtR, A, lda, Y, ldy, l, ncols, m, pw, nb, c->num_sms,
                                c->stream, piped ? &c->crt_pipe : nullptr, &tim, launches));
    c->crt_timed = tim.used;
    return RID_OK;
  }
  if (sr.strassen) {
    if (col0 % 64 != 0 || ncols % 64 != 0)
      return fail(c, RID_EINVAL,
                  "sketch: with the Strassen plan of (l=%lld, m=%lld, n=%lld) a column block must "
                  "start and end on multiples of 64 (col0=%lld, ncols=%lld); RID_SKETCH_STRASSEN=0 "
                  "selects the plain 3M sketch", (long long)l, (long long)m, (long long)n,
                  (long long)col0, (long long)ncols);
    void* pm;
    const int Sk = rid::strassen_ksplit(l, m, n, c->num_sms);
    RID_TRY(ws_get(c, "Mstr", (size_t)Sk * rid::strassen_ws(l, m, ncols).m_bytes, &pm));
    RID_CUDA(c, rid::strassen_sketch(sr.Rc, sr.sw.ldc, sr.Rsc, sr.sw.lds, A, lda, Y, ldy, l, ncols,
                                     m, (double2*)pm, Sk, c->stream, aux, launches));
    return RID_OK;
  }
  RID_CUDA(c, rid::sketch_gemm(sr.R, l, sr.Rs, A, lda, Y, ldy, l, ncols, m, c->stream, S, partial,
                               col0, n, c->num_sms, launches, aux));
  return RID_OK;
}

// Y[:, 0:n_loc] = R A for a HOST A (the e2e path): A is streamed to the device in column chunks
// of ~1 GiB on a copy stream, double-buffered, each chunk's sketch overlapping the copy of the
// next. The sketch of a column does not depend on the chunking, so Y is bit-identical to the
// device-resident call. The device never holds more than two chunks of A.
rid_status sketch_streamed(rid_ctx* c, const SketchR& sr, const rid_z* hostA,
                           int64_t m, int64_t n, int64_t col0, int64_t n_loc, int64_t lda,
                           int64_t l, double2* Y, int* launches, double* t_h2d, int ksplit,
                           double2* partial) {
  if (!c->copy_stream) {
    RID_CUDA(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      RID_CUDA(c, cudaEventCreateWithFlags(&c->ev_copied[b], cudaEventDisableTiming));
      RID_CUDA(c, cudaEventCreateWithFlags(&c->ev_used[b], cudaEventDisableTiming));
    }
    RID_CUDA(c, cudaEventCreate(&c->ev_copy0));
    RID_CUDA(c, cudaEventCreate(&c->ev_copy1));
  }
  int64_t chunk = (int64_t)(1 << 30) / (16 * m) / 64 * 64;  // whole 64-column groups
  if (chunk < 64) chunk = 64;
  if (chunk > n_loc) chunk = n_loc;
  void* buf[2];
  RID_TRY(ws_get(c, "streamA0", sizeof(double2) * m * chunk, &buf[0]));
  RID_TRY(ws_get(c, "streamA1", sizeof(double2) * m * chunk, &buf[1]));
  // the copy stream must not overwrite a buffer before the previous call's kernels used it
  RID_CUDA(c, cudaEventRecord(c->ev_used[0], c->stream));
  RID_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->ev_used[0], 0));
  RID_CUDA(c, cudaEventRecord(c->ev_copy0, c->copy_stream));
  int i = 0;
  for (int64_t j0 = 0; j0 < n_loc; j0 += chunk, ++i) {
    const int b = i & 1;
    const int64_t nc = (j0 + chunk <= n_loc) ? chunk : n_loc - j0;
    if (i >= 2) RID_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->ev_used[b], 0));
    RID_CUDA(c, cudaMemcpy2DAsync(buf[b], sizeof(double2) * m, hostA + j0 * lda,
                                  sizeof(double2) * lda, sizeof(double2) * m, nc,
                                  cudaMemcpyHostToDevice, c->copy_stream));
    RID_CUDA(c, cudaEventRecord(c->ev_copied[b], c->copy_stream));
    RID_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));
    RID_TRY(sketch_block(c, sr, (const double2*)buf[b], m, Y + j0 * l, l, l, nc, m, col0 + j0, n,
                         ksplit, partial, launches, nullptr));
    RID_CUDA(c, cudaEventRecord(c->ev_used[b], c->stream));
  }
  RID_CUDA(c, cudaEventRecord(c->ev_copy1, c->copy_stream));
  if (t_h2d) {
    RID_CUDA(c, cudaEventSynchronize(c->ev_copy1));
    *t_h2d += ev_ms(c->ev_copy0, c->ev_copy1) * 1e-3;
  }
  return RID_OK;
}

// SRFT sketch of a device A (a_dev) or a host A (host_A, staged whole) into Y (device, ldy).
rid_status srft_into(rid_ctx* c, uint64_t seed, bool retry, int64_t l, const rid_z* host_A,
                     const void* a_dev, int64_t m, int64_t n, int64_t n_loc, int64_t lda,
                     double2* Y, int64_t ldy, int* launches) {
  if (m < 16 || (m & (m - 1)) != 0)
    return fail(c, RID_EINVAL, "SRFT sketch: m = %lld must be a power of two >= 16", (long long)m);
  if (!a_dev) {
    MatArg a;
    RID_TRY(stage_in(c, "stage_A", host_A, m, n_loc, lda, sizeof(rid_z), true, &a));
    a_dev = a.dev;
  }
  void *pw, *ps;
  RID_TRY(ws_get(c, "srft_work", rid::srft_work_bytes(m, l, n_loc), &pw));
  const size_t split_elems = (size_t)8 * (size_t)l * 4096;  // bounded split-K workspace
  RID_TRY(ws_get(c, "srft_splitk", sizeof(double2) * split_elems, &ps));
  RID_CUDA(c, rid::srft_sketch(seed, retry, l, (const double2*)a_dev, m, n, n_loc, lda, Y, ldy, pw,
                               (double2*)ps, split_elems, c->num_sms, c->stream, launches));
  return RID_OK;
}

rid_status LocalComm::allreduce_sum(rid_ctx* c, double* buf, size_t count) {
  void* tmp;
  RID_TRY(ws_get(c, "comm_sum", count * sizeof(double), &tmp));
  RID_TRY(publish(c, buf));
  rid::RankPtrs src{};
  for (int h = 0; h < g->G; ++h) {
    if (h != rank) RID_CUDA(c, cudaStreamWaitEvent(c->stream, g->ready[h], 0));
    src.p[h] = g->buf[h];
  }
  RID_CUDA(c, rid::sum_ranks(src, g->G, (double*)tmp, (int64_t)count, c->stream));
  RID_TRY(finish(c));  // every peer has read buf: it may be overwritten
  RID_CUDA(c, cudaMemcpyAsync(buf, tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return RID_OK;
}

// The sharded QR on one device: every rank publishes its part; rank 0 launches the one kernel
// over all G blocks (rid::qrcp_sharded: G rank groups of CTAs in one cooperative grid, the form
// the profiling rules prescribe for more ranks than GPUs) on its stream after every rank's
// `ready`; every rank's stream then waits for rank 0's `done`.
rid_status LocalComm::qr_sharded(rid_ctx* c, const ShardQrPart& part, int* launches) {
  g->qr.resize(g->G);
  g->qr[rank] = part;
  RID_CUDA(c, cudaEventRecord(g->ready[rank], c->stream));
  RID_TRY(rendezvous(c));
  if (rank == 0) {
    rid::QrShards sh;
    sh.G = g->G;
    sh.n_loc = part.n_loc;
    rid_status st = RID_OK;
    for (int h = 0; h < g->G; ++h) {
      const ShardQrPart& q = g->qr[h];
      if (q.n_loc != part.n_loc || q.l != part.l || q.k != part.k || q.ldy != part.ldy)
        st = RID_EINVAL;
      sh.Y[h] = q.Y;
      sh.out[h] = q.out;
      sh.w[h] = q.w;
      if (h != rank) {
        cudaError_t e = cudaStreamWaitEvent(c->stream, g->ready[h], 0);
        if (e != cudaSuccess) st = RID_ECUDA;
      }
    }
    g->qr_err.clear();
    if (st == RID_OK) {
      const cudaError_t e = rid::qrcp_sharded(sh, part.ldy, part.l, part.k, part.tol, c->num_sms,
                                              c->stream, launches);
      if (e != cudaSuccess) {
        st = RID_ECUDA;
        g->qr_err = cudaGetErrorString(e);
      }
    } else if (g->qr_err.empty()) {
      g->qr_err = "ranks disagree on (l, k, n_loc, ldy)";
    }
    g->qr_status = st;
  }
  RID_TRY(finish(c));  // every rank's stream now waits for rank 0's done (after the kernel)
  if (g->qr_status != RID_OK)
    return fail(c, g->qr_status, "sharded QR (rank 0): %s", g->qr_err.c_str());
  return RID_OK;
}

__global__ void k_extract_R(const double2* __restrict__ Y, int64_t ldy, const int64_t* __restrict__ J,
                            const double2* __restrict__ R11, int64_t k, int64_t n,
                            double2* __restrict__ R, int64_t ldr) {
  // R[:, c] = Y[0:k, c] for non-pivot c; for c = J[s]: column s of the dense triangle R11
  const int64_t c = blockIdx.x;
  __shared__ int64_t s_piv;
  if (threadIdx.x == 0) {
    s_piv = -1;
    for (int64_t s = 0; s < k; ++s)
      if (J[s] == c) s_piv = s;
  }
  __syncthreads();
  const int64_t s = s_piv;
  for (int64_t t = threadIdx.x; t < k; t += blockDim.x)
    R[c * ldr + t] = (s >= 0) ? R11[s * k + t] : Y[c * ldy + t];
}

}  // namespace

extern "C" {

const char* rid_version(void) { return "librid 0.1 (sm_100a, DMMA fp64 tensor pipe)"; }

rid_status rid_create(rid_ctx** out, int device, void* cuda_stream) {
  if (!out) return RID_EINVAL;
  *out = nullptr;
  rid_ctx* c = new rid_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete c;
    return RID_ECUDA;
  }
  c->stream = (cudaStream_t)cuda_stream;  // NULL = the legacy default stream, as in CUDA
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  *out = c;
  return RID_OK;
}

rid_status rid_set_stream(rid_ctx* c, void* cuda_stream) {
  RID_TRY(check_ctx(c));
  if (c->owns_stream && c->stream != (cudaStream_t)cuda_stream) {
    RID_CUDA(c, cudaStreamSynchronize(c->stream));
    RID_CUDA(c, cudaStreamDestroy(c->stream));
    c->owns_stream = false;
  }
  c->stream = (cudaStream_t)cuda_stream;
  return RID_OK;
}

void rid_destroy(rid_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->ws)
    if (kv.second.p) cudaFree(kv.second.p);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  c->comm.reset();
  if (c->host_qr) cudaFreeHost(c->host_qr);
  if (c->aux_stream) {
    cudaStreamSynchronize(c->aux_stream);
    cudaStreamDestroy(c->aux_stream);
    cudaEventDestroy(c->aux_fork);
    cudaEventDestroy(c->aux_join);
  }
  for (auto& e : c->crt_tev)
    if (e) cudaEventDestroy(e);
  if (c->crt_pipe.stream) {
    cudaStreamSynchronize(c->crt_pipe.stream);
    cudaStreamDestroy(c->crt_pipe.stream);
    cudaEvent_t* evs[6] = {&c->crt_pipe.fork, &c->crt_pipe.join, &c->crt_pipe.prep[0],
                           &c->crt_pipe.prep[1], &c->crt_pipe.gemm[0], &c->crt_pipe.gemm[1]};
    for (auto* e : evs) cudaEventDestroy(*e);
  }
  if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
  if (c->cap_stream) {
    cudaStreamSynchronize(c->cap_stream);
    cudaStreamDestroy(c->cap_stream);
    cudaEventDestroy(c->g_in);
    cudaEventDestroy(c->g_out);
  }
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(c->ev_copied[b]);
      cudaEventDestroy(c->ev_used[b]);
    }
    cudaEventDestroy(c->ev_copy0);
    cudaEventDestroy(c->ev_copy1);
  }
  if (c->owns_stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* rid_last_error(const rid_ctx* c) { return c ? c->err.c_str() : "null context"; }

size_t rid_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

rid_status rid_comm_get_id(void* id) {
  if (!id) return RID_EINVAL;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return RID_ENCCL;
  std::memcpy(id, &u, sizeof u);
  return RID_OK;
}

rid_status rid_comm_init(rid_ctx* c, const void* id, int rank, int nranks) {
  RID_TRY(check_ctx(c));
  if (!id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(c, RID_EINVAL, "rid_comm_init: bad rank %d / nranks %d", rank, nranks);
  c->comm.reset();
  c->rank = 0;
  c->nranks = 1;
  // a 1-rank communicator is created only on request (RID_FORCE_NCCL=1): it routes a single
  // GPU through the collective code path (tests/test_gpu_collective.py)
  if (nranks > 1 || rid::select_env("RID_FORCE_NCCL")) {
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    auto nc = std::make_unique<NcclComm>();
    RID_NCCL(c, ncclCommInitRank(&nc->comm, nranks, u, rank));
    nc->rank = rank;
    nc->nranks = nranks;
    c->comm = std::move(nc);
  }
  c->rank = rank;
  c->nranks = nranks;
  return RID_OK;
}

rid_status rid_comm_init_local(rid_ctx** ctxs, int nranks) {
  if (!ctxs || nranks < 1 || nranks > rid::kMaxLocalRanks) return RID_EINVAL;
  for (int r = 0; r < nranks; ++r) {
    if (!ctxs[r]) return RID_EINVAL;
    for (int h = 0; h < r; ++h)
      if (ctxs[h] == ctxs[r]) return fail(ctxs[r], RID_EINVAL, "rid_comm_init_local: context repeated");
    if (ctxs[r]->device != ctxs[0]->device)
      return fail(ctxs[r], RID_EINVAL, "rid_comm_init_local: all contexts must be on one device");
  }
  rid_ctx* c = ctxs[0];
  RID_TRY(check_ctx(c));
  auto g = std::make_shared<LocalGroup>();
  g->G = nranks;
  g->device = c->device;
  g->buf.assign(nranks, nullptr);
  g->ready.assign(nranks, nullptr);
  g->done.assign(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    RID_CUDA(c, cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming));
    RID_CUDA(c, cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming));
  }
  for (int r = 0; r < nranks; ++r) {
    auto lc = std::make_unique<LocalComm>();
    lc->g = g;
    lc->rank = r;
    lc->nranks = nranks;
    ctxs[r]->comm = std::move(lc);
    ctxs[r]->rank = r;
    ctxs[r]->nranks = nranks;
  }
  return RID_OK;
}

rid_status rid_comm_info(const rid_ctx* c, int* rank, int* nranks) {
  if (!c) return RID_EINVAL;
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  return RID_OK;
}

double rid_error_bound(int64_t m, int64_t n, int64_t k, double eps, double sigma_kp1) {
  if (m < 1 || n < 1 || k < 1 || !(eps > 0.0) || eps > 1.0) return NAN;
  return 50.0 * std::sqrt((double)m * (double)n) * std::pow(1.0 / eps, 1.0 / (double)k) * sigma_kp1;
}

rid_status rid_normal_fill(rid_ctx* c, uint64_t seed, uint32_t s, int64_t rows, int64_t cols,
                           int64_t row0, int64_t col0, rid_z* out, int64_t ld) {
  RID_TRY(check_ctx(c));
  if (rows < 0 || cols < 0 || row0 < 0 || col0 < 0 || ld < rows || !out ||
      row0 + rows > (int64_t)0xFFFFFFFFLL || col0 + cols > (int64_t)0xFFFFFFFFLL)
    return fail(c, RID_EINVAL, "rid_normal_fill: bad shape");
  MatArg o;
  RID_TRY(stage_in(c, "stage_out0", out, rows, cols, ld, sizeof(rid_z), false, &o));
  RID_CUDA(c, rid::normal_fill(seed, s, rows, cols, row0, col0, (double2*)o.dev, ld, c->stream));
  RID_TRY(stage_out(c, o, out, rows, cols, ld, sizeof(rid_z)));
  if (o.host) RID_CUDA(c, cudaStreamSynchronize(c->stream));
  return RID_OK;
}

rid_status rid_generate(rid_ctx* c, uint64_t seed, int64_t m, int64_t n, int64_t k, double noise,
                        int64_t col0, int64_t n_loc, rid_z* A, int64_t lda) {
  RID_TRY(check_ctx(c));
  if (m < 1 || n < 1 || k < 1 || k > m || k > n || col0 < 0 || n_loc < 0 || col0 + n_loc > n ||
      lda < m || !A || m > (int64_t)0xFFFFFFFFLL || n > (int64_t)0xFFFFFFFFLL || !std::isfinite(noise))
    return fail(c, RID_EINVAL, "rid_generate: bad arguments (m=%lld n=%lld k=%lld col0=%lld n_loc=%lld lda=%lld)",
                (long long)m, (long long)n, (long long)k, (long long)col0, (long long)n_loc, (long long)lda);
  if (n_loc == 0) return RID_OK;
  MatArg a;
  RID_TRY(stage_in(c, "stage_A", A, m, n_loc, lda, sizeof(rid_z), false, &a));
  void *pX, *pY0;
  RID_TRY(ws_get(c, "X", sizeof(double2) * m * k, &pX));
  RID_TRY(ws_get(c, "Y0", sizeof(double2) * k * n_loc, &pY0));
  RID_CUDA(c, rid::normal_fill(seed, 1u, m, k, 0, 0, (double2*)pX, m, c->stream));
  RID_CUDA(c, rid::normal_fill(seed, 2u, k, n_loc, 0, col0, (double2*)pY0, k, c->stream));
  RID_CUDA(c, rid::zgemm_ordered((const double2*)pX, m, (const double2*)pY0, k, (double2*)a.dev, lda,
                                 m, n_loc, k, noise != 0.0 ? 1 : 0, noise, seed, col0, c->stream));
  RID_TRY(stage_out(c, a, A, m, n_loc, lda, sizeof(rid_z)));
  if (a.host) RID_CUDA(c, cudaStreamSynchronize(c->stream));
  return RID_OK;
}

rid_status rid_set_sketch(rid_ctx* c, int kind) {
  if (!c) return RID_EINVAL;
  if (kind != RID_SKETCH_GAUSSIAN && kind != RID_SKETCH_SRFT)
    return fail(c, RID_EINVAL, "rid_set_sketch: unknown kind %d", kind);
  c->sketch_kind = kind;
  return RID_OK;
}

rid_status rid_set_sketch_engine(rid_ctx* c, int engine) {
  if (!c) return RID_EINVAL;
  if (engine != RID_ENGINE_AUTO && engine != RID_ENGINE_FP64_DMMA && engine != RID_ENGINE_INT8_CRT)
    return fail(c, RID_EINVAL, "rid_set_sketch_engine: unknown engine %d", engine);
  c->sketch_engine = engine;
  return RID_OK;
}

int rid_sketch_engine_of(const rid_ctx* c, int64_t m, int64_t l, int64_t n) {
  if (!c || m < 1 || l < 1 || n < 1) return 0;
  return use_crt(c, l, m, n) ? RID_ENGINE_INT8_CRT : RID_ENGINE_FP64_DMMA;
}

rid_status rid_crt_plan(int64_t l, int64_t m, int* T, int* b, int* kslices, int64_t* Kp, int* nc,
                        double* log2M) {
  if (l < 1 || m < 1 || l > 2048) return RID_EINVAL;
  const rid::CrtPlan p = rid::crt_plan(l, m);
  if (T) *T = p.T;
  if (b) *b = p.b;
  if (kslices) *kslices = p.kslices;
  if (Kp) *Kp = p.Kp;
  if (nc) *nc = p.nc;
  if (log2M) *log2M = rid::crt_log2M(p.T);
  return RID_OK;
}

int rid_crt_moduli(int* p, int cap) { return rid::crt_moduli(p, cap); }

rid_status rid_set_qr_dist(rid_ctx* c, int mode) {
  if (!c) return RID_EINVAL;
  if (mode != RID_QR_REPLICATED && mode != RID_QR_SHARDED)
    return fail(c, RID_EINVAL, "rid_set_qr_dist: unknown mode %d", mode);
  c->qr_dist = mode;
  return RID_OK;
}

rid_status rid_set_qr(rid_ctx* c, int kind) {
  if (!c) return RID_EINVAL;
  if (kind != RID_QR_HOUSEHOLDER && kind != RID_QR_CGS2)
    return fail(c, RID_EINVAL, "rid_set_qr: unknown kind %d", kind);
  c->qr_kind = kind;
  return RID_OK;
}

rid_status rid_sketch_srft(rid_ctx* c, uint64_t seed, int retry, int64_t l, const rid_z* A,
                           int64_t m, int64_t n, int64_t n_loc, int64_t lda, rid_z* Y,
                           int64_t ldy) {
  RID_TRY(check_ctx(c));
  if (l < 1 || m < 16 || (m & (m - 1)) != 0 || n_loc < 0 || n < n_loc || lda < m || ldy < l ||
      !A || !Y || m > (int64_t)0xFFFFFFFFLL || n_loc > 0xFFFFFFFFLL)
    return fail(c, RID_EINVAL, "rid_sketch_srft: bad arguments (m must be a power of two >= 16)");
  if (n_loc == 0) return RID_OK;
  MatArg a, y;
  RID_TRY(stage_in(c, "stage_A", A, m, n_loc, lda, sizeof(rid_z), true, &a));
  RID_TRY(stage_in(c, "stage_Y", Y, l, n_loc, ldy, sizeof(rid_z), false, &y));
  int launches = 0;
  RID_TRY(srft_into(c, seed, retry != 0, l, nullptr, a.dev, m, n, n_loc, lda, (double2*)y.dev, ldy,
                    &launches));
  RID_TRY(stage_out(c, y, Y, l, n_loc, ldy, sizeof(rid_z)));
  if (a.host || y.host) RID_CUDA(c, cudaStreamSynchronize(c->stream));
  return RID_OK;
}

int rid_sketch_splits(const rid_ctx* c, int64_t m, int64_t l, int64_t n) {
  if (!c || m < 1 || l < 1 || n < 1) return 1;
  return rid::sketch_ksplit(l, m, n / 8, c->num_sms);
}

int rid_sketch_mults(void) { return rid::sketch_mults(); }

int rid_sketch_strassen(const rid_ctx* c, int64_t m, int64_t l, int64_t n) {
  if (!c || m < 1 || l < 1 || n < 1) return 0;
  return strassen_on(c, l, m, n) ? 1 : 0;
}

rid_status rid_sketch(rid_ctx* c, uint64_t seed, uint32_t stream, int64_t l, const rid_z* A,
                      int64_t m, int64_t n, int64_t n_loc, int64_t lda, rid_z* Y, int64_t ldy) {
  return rid_sketch_cols(c, seed, stream, l, A, m, n, 0, n_loc, lda, Y, ldy);
}

rid_status rid_sketch_cols(rid_ctx* c, uint64_t seed, uint32_t stream, int64_t l, const rid_z* A,
                           int64_t m, int64_t n, int64_t col0, int64_t n_loc, int64_t lda, rid_z* Y,
                           int64_t ldy) {
  RID_TRY(check_ctx(c));
  if (l < 1 || l > m || m < 1 || n_loc < 0 || col0 < 0 || col0 + n_loc > n || lda < m ||
      ldy < l || !A || !Y || m > (int64_t)0xFFFFFFFFLL)
    return fail(c, RID_EINVAL, "rid_sketch: bad arguments");
  if (n_loc == 0) return RID_OK;
  MatArg a, y;
  RID_TRY(stage_in(c, "stage_A", A, m, n_loc, lda, sizeof(rid_z), true, &a));
  RID_TRY(stage_in(c, "stage_Y", Y, l, n_loc, ldy, sizeof(rid_z), false, &y));
  void* pS = nullptr;
  SketchR sr;
  int nl = 0;
  if (strassen_on(c, l, m, n) && (col0 % 64 != 0 || n_loc % 64 != 0))
    return fail(c, RID_EINVAL, "rid_sketch: with the Strassen plan of this (l, m, n) a column "
                               "block must start and end on multiples of 64");
  RID_TRY(fill_R(c, seed, stream, l, m, n, &sr, &nl));
  const int S = rid::sketch_ksplit(l, m, n / 8, c->num_sms);
  const int64_t pe = sr.strassen ? 0 : rid::sketch_partial_elems(l, m, n, n_loc, c->num_sms);
  if (pe > 0) RID_TRY(ws_get(c, "splitk", sizeof(double2) * pe, &pS));
  rid::SketchAux auxv;
  const rid::SketchAux* aux = nullptr;
  if (sr.strassen) RID_TRY(sketch_aux(c, &auxv, &aux));  // the row split of the products
  RID_TRY(sketch_block(c, sr, (const double2*)a.dev, lda, (double2*)y.dev, ldy, l, n_loc, m, col0,
                       n, S, (double2*)pS, &nl, aux));
  RID_TRY(stage_out(c, y, Y, l, n_loc, ldy, sizeof(rid_z)));
  if (a.host || y.host) RID_CUDA(c, cudaStreamSynchronize(c->stream));
  return RID_OK;
}

rid_status rid_decompose(rid_ctx* c, const rid_z* A, int64_t m, int64_t n, int64_t col0,
                         int64_t n_loc, int64_t lda, int64_t k, int64_t l, uint64_t seed,
                         int64_t* J, rid_z* P, int64_t ldp, rid_diag* diag) {
  RID_TRY(check_ctx(c));
  if (m < 1 || n < 1 || k < 1 || k > m || k > n || l < k || l > m || l > 2048 || col0 < 0 ||
      n_loc < 1 || col0 + n_loc > n || lda < m || ldp < k || !A || !J || !P ||
      m > (int64_t)0xFFFFFFFFLL)
    return fail(c, RID_EINVAL, "rid_decompose: bad arguments (m=%lld n=%lld k=%lld l=%lld col0=%lld n_loc=%lld)",
                (long long)m, (long long)n, (long long)k, (long long)l, (long long)col0, (long long)n_loc);
  if (c->nranks > 1 && (n_loc * c->nranks != n || col0 != n_loc * c->rank))
    return fail(c, RID_EINVAL, "rid_decompose: shard (%lld, %lld) is not rank %d's 1/%d of n=%lld",
                (long long)col0, (long long)n_loc, c->rank, c->nranks, (long long)n);
  if (c->nranks == 1 && (col0 != 0 || n_loc != n))
    return fail(c, RID_EINVAL, "rid_decompose: without a communicator the shard must be all of A");
  // sharded QR (NEXT-3): Householder only, on a data plane that has it, equal shards
  const bool sharded = c->comm && c->qr_dist == RID_QR_SHARDED && c->comm->has_sharded_qr() &&
                       c->qr_kind == RID_QR_HOUSEHOLDER;
  if (c->comm && c->qr_dist == RID_QR_SHARDED && !sharded)
    return fail(c, RID_EINVAL, "rid_decompose: RID_QR_SHARDED needs the Householder QR and a "
                               "communicator with a sharded QR (rid_comm_init_local, <= %d ranks)",
                rid::kQrMaxRanks);
  rid_diag d{};
  cudaEvent_t* ev = c->ev;
  RID_CUDA(c, cudaEventRecord(ev[0], c->stream));
  MatArg a, p;
  const bool a_host = !is_device_ptr(A);  // host A is streamed chunk by chunk under the sketch
  if (!a_host) RID_TRY(stage_in(c, "stage_A", A, m, n_loc, lda, sizeof(rid_z), true, &a));
  RID_TRY(stage_in(c, "stage_P", P, k, n_loc, ldp, sizeof(rid_z), false, &p));
  RID_CUDA(c, cudaEventRecord(ev[1], c->stream));
  void *pY, *pR;
  RID_TRY(ws_get(c, "Y", sizeof(double2) * l * n, &pY));
  RID_TRY(ws_get(c, "R", sizeof(double2) * l * m, &pR));
  double2* Yw = (double2*)pY;
  // K-split of the sketch: a function of (m, l, n) only, so Y is identical for every sharding
  const int S = rid::sketch_ksplit(l, m, n / 8, c->num_sms);
  const bool strassen = c->sketch_kind != RID_SKETCH_SRFT && strassen_on(c, l, m, n);
  if (strassen && (col0 % 64 != 0 || n_loc % 64 != 0))
    return fail(c, RID_EINVAL, "rid_decompose: with the Strassen sketch plan of this (l, m, n) a "
                               "shard must start and end on multiples of 64 columns");
  void* pS = nullptr;
  if (!strassen) {
    const int64_t cols = a_host ? std::min<int64_t>(n_loc, std::max<int64_t>(64, (int64_t)(1 << 30) / (16 * m)))
                                : n_loc;
    const int64_t pe = rid::sketch_partial_elems(l, m, n, cols, c->num_sms);
    if (pe > 0) RID_TRY(ws_get(c, "splitk", sizeof(double2) * pe, &pS));
  }
  int64_t* Jdev = nullptr;
  rid_status st = RID_OK;
  int info[2] = {0, 0};
  const bool j_dev = is_device_ptr(J);
  // the device work of one attempt (events ev[2]..ev[8], R, sketch, all-gather, QR, its status
  // copy, solve, J): enqueue only, no synchronisation
  // ev[2..8]: while capturing, recorded as external events, so inside the graph they stay real
  // event records the host can synchronise on and time (the flag is refused outside capture)
  bool capturing = false;
  auto rec = [&](cudaEvent_t e) {
    return capturing ? cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal)
                     : cudaEventRecord(e, c->stream);
  };
  auto enqueue = [&](int attempt) -> rid_status {
    const uint32_t sR = attempt == 0 ? kStreamR : kStreamRRetry;
    RID_CUDA(c, rec(ev[2]));
    if (c->sketch_kind == RID_SKETCH_SRFT) {  // the paper's own randomisation
      RID_CUDA(c, rec(ev[3]));
      RID_TRY(srft_into(c, seed, attempt == 1, l, A, a_host ? nullptr : a.dev, m, n, n_loc, lda,
                        Yw + col0 * l, l, &d.launches));
    } else {
    SketchR sr;
    RID_TRY(fill_R(c, seed, sR, l, m, n, &sr, &d.launches));
    RID_CUDA(c, rec(ev[3]));
    if (a_host) {
      RID_TRY(sketch_streamed(c, sr, A, m, n, col0, n_loc, lda, l, Yw + col0 * l, &d.launches,
                              nullptr, S, (double2*)pS));
    } else {
      rid::SketchAux auxv;
      const rid::SketchAux* aux = nullptr;
      RID_TRY(sketch_aux(c, &auxv, &aux));
      RID_TRY(sketch_block(c, sr, (const double2*)a.dev, lda, Yw + col0 * l, l, l, n_loc, m, col0,
                           n, S, (double2*)pS, &d.launches, aux));
    }
    }
    RID_CUDA(c, rec(ev[4]));
    if (c->comm && !sharded) RID_TRY(c->comm->allgather(c, (double*)Yw, (size_t)(2 * l * n_loc)));
    RID_CUDA(c, rec(ev[5]));
    // the QR, its status copy and the solve are enqueued together; the status is checked after
    // the one synchronisation at the end (a failed attempt's solve output is discarded).
    // Sharded (NEXT-3): no all-gather; this rank's block is factored with the others' in place.
    if (sharded)
      RID_TRY(factor_and_solve(c, Yw + col0 * l, l, n_loc, k, 0, n_loc, (double2*)p.dev, ldp,
                               &Jdev, info, &d, false, nullptr, /*defer=*/true, /*sharded=*/true));
    else
      RID_TRY(factor_and_solve(c, Yw, l, n, k, col0, n_loc, (double2*)p.dev, ldp, &Jdev, info, &d,
                               false, nullptr, /*defer=*/true));
    RID_CUDA(c, rec(ev[6]));
    {  // solve
      void *pR11, *pRinv;
      RID_TRY(ws_get(c, "R11", sizeof(double2) * k * k, &pR11));
      RID_TRY(ws_get(c, "Rinv", sizeof(double2) * k * k, &pRinv));
      RID_CUDA(c, rid::tri_inverse((const double2*)pR11, k, (double2*)pRinv, c->stream));
      RID_TRY(solve_T(c, (const double2*)pRinv, k, Yw + col0 * l, l, (double2*)p.dev, ldp, n_loc,
                      &d.launches, c->sketch_kind != RID_SKETCH_SRFT && use_crt(c, l, m, n)));
      RID_CUDA(c, rid::assemble_identity(Jdev, k, col0, n_loc, (double2*)p.dev, ldp, c->stream));
      d.launches += 2;  // R11^-1, identity (solve_T counts the sum plane and the T GEMM)
    }
    RID_CUDA(c, rec(ev[7]));
    RID_TRY(stage_out(c, p, P, k, n_loc, ldp, sizeof(rid_z)));
    if (j_dev)
      RID_CUDA(c, cudaMemcpyAsync(J, Jdev, sizeof(int64_t) * k, cudaMemcpyDeviceToDevice, c->stream));
    else
      RID_CUDA(c, cudaMemcpyAsync(J, Jdev, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, c->stream));
    RID_CUDA(c, rec(ev[8]));
    return RID_OK;
  };
  // repeated calls with identical arguments replay a CUDA graph of that work (one launch instead
  // of ~30 API calls: the small configs are launch-bound); captured on the second such call,
  // device A / J / P and no communicator only, RID_GRAPH=0 disables; any capture failure falls
  // back to the eager path
  const bool graphable = !a_host && !p.host && j_dev && !c->comm &&
                         c->sketch_kind != RID_SKETCH_SRFT &&
                         !(rid::select_env("RID_GRAPH") && atoi(rid::select_env("RID_GRAPH")) == 0);
  std::string gkey;
  if (graphable) {
    char buf[512];
    snprintf(buf, sizeof buf, "%p %lld %lld %lld %lld %lld %lld %lld %llu %p %p %lld %d %llu %p %d",
             (const void*)A, (long long)m, (long long)n, (long long)col0, (long long)n_loc,
             (long long)lda, (long long)k, (long long)l, (unsigned long long)seed, (void*)J,
             (void*)p.dev, (long long)ldp, c->qr_kind, c->ws_epoch, c->host_qr, c->sketch_engine);
    gkey = buf;
    for (char** e = environ; *e; ++e)  // every RID_* knob selects kernels: part of the key
      if (strncmp(*e, "RID_", 4) == 0) {
        gkey += ' ';
        gkey += *e;
      }
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    bool replayed = false;
    if (attempt == 0 && graphable) {
      if (!c->cap_stream) {
        RID_CUDA(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        RID_CUDA(c, cudaEventCreateWithFlags(&c->g_in, cudaEventDisableTiming));
        RID_CUDA(c, cudaEventCreateWithFlags(&c->g_out, cudaEventDisableTiming));
      }
      if (!(c->g_exec && c->g_key == gkey) && c->g_seen == gkey && c->g_bad != gkey) {  // capture
        cudaStream_t orig = c->stream;
        c->stream = c->cap_stream;
        const int l0 = d.launches;
        cudaGraph_t g = nullptr;
        rid_status es = RID_ECUDA;
        if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
          capturing = c->capturing = true;
          es = enqueue(0);
          capturing = c->capturing = false;
          c->g_crt_timed = c->crt_timed;
          if (cudaStreamEndCapture(c->cap_stream, &g) != cudaSuccess) es = RID_ECUDA;
        }
        c->stream = orig;
        cudaGraphExec_t ex = nullptr;
        if (es == RID_OK && g && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
          if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
          c->g_exec = ex;
          c->g_key = gkey;
          c->g_launches = d.launches - l0;
        } else {
          c->g_bad = gkey;  // not capturable: stay eager for these arguments
        }
        if (rid::select_env("RID_GRAPH_DEBUG"))
          fprintf(stderr, "rid_decompose: graph capture %s (%s; %s)\n",
                  c->g_key == gkey ? "ok" : "FAILED", es == RID_OK ? "enqueue ok" : c->err.c_str(),
                  cudaGetErrorString(cudaGetLastError()));
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();  // a failed capture leaves no sticky error: the eager path follows
        d.launches = l0;
        c->err.clear();
      }
      if (c->g_exec && c->g_key == gkey) {
        RID_CUDA(c, cudaEventRecord(c->g_in, c->stream));
        RID_CUDA(c, cudaStreamWaitEvent(c->cap_stream, c->g_in, 0));
        RID_CUDA(c, cudaGraphLaunch(c->g_exec, c->cap_stream));
        c->crt_timed = c->g_crt_timed;
        RID_CUDA(c, cudaEventRecord(c->g_out, c->cap_stream));
        RID_CUDA(c, cudaStreamWaitEvent(c->stream, c->g_out, 0));
        d.launches += c->g_launches;
        replayed = true;
      }
      c->g_seen = gkey;
    }
    if (!replayed) RID_TRY(enqueue(attempt));
    RID_CUDA(c, cudaEventSynchronize(ev[8]));
    st = qr_check(c, k, info, &d);
    if (st == RID_ERANK && attempt == 0) {
      d.retries = 1;
      continue;  // repeat with a different instance of the random matrix
    }
    break;
  }
  if (st == RID_ERANK) {
    if (diag) *diag = d;
    return fail(c, RID_ERANK, "sketch rank %d < k = %lld after one re-randomisation", d.rank_achieved,
                (long long)k);
  }
  if (st != RID_OK) return st;
  if (diag) {
    // host A: the streamed copies overlap the sketch (t_sketch then includes copy stalls)
    d.t_h2d = a_host ? ev_ms(c->ev_copy0, c->ev_copy1) * 1e-3 : ev_ms(ev[0], ev[1]) * 1e-3;
    d.t_rgen = ev_ms(ev[2], ev[3]) * 1e-3;
    d.t_sketch = ev_ms(ev[3], ev[4]) * 1e-3;
    d.t_gather = ev_ms(ev[4], ev[5]) * 1e-3;
    d.t_qrcp = ev_ms(ev[5], ev[6]) * 1e-3;
    d.t_solve = ev_ms(ev[6], ev[7]) * 1e-3;
    d.t_d2h = ev_ms(ev[7], ev[8]) * 1e-3;
    d.t_total = ev_ms(ev[0], ev[8]) * 1e-3;
    d.sketch_engine = 0;
    d.t_sketch_tc = 0.0;
    if (c->sketch_kind != RID_SKETCH_SRFT) {
      d.sketch_engine = use_crt(c, l, m, n) ? RID_ENGINE_INT8_CRT : RID_ENGINE_FP64_DMMA;
      if (d.sketch_engine == RID_ENGINE_INT8_CRT)
        for (int g = 0; g < c->crt_timed; ++g)
          d.t_sketch_tc += ev_ms(c->crt_tev[2 * g], c->crt_tev[2 * g + 1]) * 1e-3;
    }
    *diag = d;
  }
  return RID_OK;
}

rid_status rid_qrcp(rid_ctx* c, const rid_z* Y, int64_t l, int64_t n, int64_t ldy, int64_t k,
                    int64_t* J, rid_z* R, int64_t ldr, double* resid, double* margin,
                    rid_diag* diag) {
  RID_TRY(check_ctx(c));
  if (l < 1 || n < 1 || k < 1 || k > l || k > n || l > 2048 || ldy < l || !Y || !J ||
      (R && ldr < k))
    return fail(c, RID_EINVAL, "rid_qrcp: bad arguments");
  MatArg y;
  RID_TRY(stage_in(c, "stage_Yin", Y, l, n, ldy, sizeof(rid_z), true, &y));
  void* pY;
  RID_TRY(ws_get(c, "Y", sizeof(double2) * l * n, &pY));
  RID_CUDA(c, cudaMemcpy2DAsync(pY, sizeof(double2) * l, y.dev, sizeof(double2) * ldy,
                                sizeof(double2) * l, n, cudaMemcpyDeviceToDevice, c->stream));
  int64_t* Jdev = nullptr;
  int info[2];
  rid_diag d{};
  double* beta = nullptr;
  rid_status st = factor_and_solve(c, (double2*)pY, l, n, k, 0, n, nullptr, k, &Jdev, info, &d,
                                   false, &beta);
  if (diag) *diag = d;
  if (st != RID_OK) return st;
  const bool jdev = is_device_ptr(J);
  RID_CUDA(c, cudaMemcpyAsync(J, Jdev, sizeof(int64_t) * k,
                              jdev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  if (R) {
    MatArg r;
    RID_TRY(stage_in(c, "stage_R", R, k, n, ldr, sizeof(rid_z), false, &r));
    void* pR11;
    RID_TRY(ws_get(c, "R11", sizeof(double2) * k * k, &pR11));
    k_extract_R<<<(unsigned)n, 128, 0, c->stream>>>((const double2*)pY, l, Jdev,
                                                     (const double2*)pR11, k, n, (double2*)r.dev,
                                                     ldr);
    RID_CUDA(c, cudaGetLastError());
    RID_TRY(stage_out(c, r, R, k, n, ldr, sizeof(rid_z)));
  }
  void* pstat;  // the status block factor_and_solve filled: info | beta | resid | margin
  RID_TRY(ws_get(c, "qr_status", 16 + 3 * sizeof(double) * (size_t)k, &pstat));
  const double* presid = (const double*)((const char*)pstat + 16) + k;
  const double* pmargin = presid + k;
  if (resid)
    RID_CUDA(c, cudaMemcpyAsync(resid, presid, sizeof(double) * k, cudaMemcpyDefault, c->stream));
  if (margin)
    RID_CUDA(c, cudaMemcpyAsync(margin, pmargin, sizeof(double) * k, cudaMemcpyDefault, c->stream));
  RID_CUDA(c, cudaStreamSynchronize(c->stream));
  return RID_OK;
}

rid_status rid_factor_solve(rid_ctx* c, const rid_z* Y, int64_t l, int64_t n, int64_t ldy,
                            int64_t k, int64_t col0, int64_t n_loc, int64_t* J, rid_z* P,
                            int64_t ldp, rid_diag* diag) {
  RID_TRY(check_ctx(c));
  if (l < 1 || n < 1 || k < 1 || k > l || k > n || l > 2048 || ldy < l || !Y || !J || !P ||
      col0 < 0 || n_loc < 1 || col0 + n_loc > n || ldp < k)
    return fail(c, RID_EINVAL, "rid_factor_solve: bad arguments");
  MatArg y, p;
  RID_TRY(stage_in(c, "stage_Yin", Y, l, n, ldy, sizeof(rid_z), true, &y));
  RID_TRY(stage_in(c, "stage_P", P, k, n_loc, ldp, sizeof(rid_z), false, &p));
  void* pY;
  RID_TRY(ws_get(c, "Y", sizeof(double2) * l * n, &pY));
  RID_CUDA(c, cudaMemcpy2DAsync(pY, sizeof(double2) * l, y.dev, sizeof(double2) * ldy,
                                sizeof(double2) * l, n, cudaMemcpyDeviceToDevice, c->stream));
  int64_t* Jdev = nullptr;
  int info[2];
  rid_diag d{};
  rid_status st = factor_and_solve(c, (double2*)pY, l, n, k, col0, n_loc, (double2*)p.dev, ldp,
                                   &Jdev, info, &d, true, nullptr);
  if (diag) *diag = d;
  if (st != RID_OK) return st;
  RID_TRY(stage_out(c, p, P, k, n_loc, ldp, sizeof(rid_z)));
  RID_CUDA(c, cudaMemcpyAsync(J, Jdev, sizeof(int64_t) * k, cudaMemcpyDefault, c->stream));
  RID_CUDA(c, cudaStreamSynchronize(c->stream));
  return RID_OK;
}

rid_status rid_error_estimate(rid_ctx* c, const rid_z* A, int64_t m, int64_t n, int64_t col0,
                              int64_t n_loc, int64_t lda, const int64_t* J, int64_t k,
                              const rid_z* P, int64_t ldp, int q, uint64_t seed, double* est,
                              rid_diag* diag) {
  RID_TRY(check_ctx(c));
  if (m < 1 || n < 1 || k < 1 || k > n || col0 < 0 || n_loc < 1 || col0 + n_loc > n || lda < m ||
      ldp < k || q < 1 || !A || !J || !P || !est || n > (int64_t)0xFFFFFFFFLL)
    return fail(c, RID_EINVAL, "rid_error_estimate: bad arguments");
  if (c->nranks > 1 && (n_loc * c->nranks != n || col0 != n_loc * c->rank))
    return fail(c, RID_EINVAL, "rid_error_estimate: shard is not rank %d's 1/%d", c->rank, c->nranks);
  if (c->nranks == 1 && (col0 != 0 || n_loc != n))
    return fail(c, RID_EINVAL, "rid_error_estimate: without a communicator the shard must be all of A");
  const int G = c->nranks;
  const bool coll = c->comm != nullptr;  // collective path (G > 1, or forced for testing)
  cudaEvent_t* ev = c->ev;
  RID_CUDA(c, cudaEventRecord(ev[0], c->stream));
  MatArg a, p;
  RID_TRY(stage_in(c, "stage_A", A, m, n_loc, lda, sizeof(rid_z), true, &a));
  RID_TRY(stage_in(c, "stage_P", P, k, n_loc, ldp, sizeof(rid_z), true, &p));
  void *pJ, *pB, *px, *pz, *py, *pu, *psb, *ppx, *pax, *pwall, *pnp, *pnn, *pest;
  RID_TRY(ws_get(c, "estJ", sizeof(int64_t) * k, &pJ));
  RID_CUDA(c, cudaMemcpyAsync(pJ, J, sizeof(int64_t) * k, cudaMemcpyDefault, c->stream));
  const rid::EstPlan pl = rid::est_plan(m, n_loc, k, c->num_sms);
  RID_TRY(ws_get(c, "estB", sizeof(double2) * m * k, &pB));
  RID_TRY(ws_get(c, "estx", sizeof(double2) * n_loc, &px));
  RID_TRY(ws_get(c, "estz", sizeof(double2) * n_loc, &pz));
  RID_TRY(ws_get(c, "esty", sizeof(double2) * m, &py));
  RID_TRY(ws_get(c, "estu", sizeof(double) * 4 * k * G, &pu));
  RID_TRY(ws_get(c, "estsb", sizeof(double) * 4 * k, &psb));
  RID_TRY(ws_get(c, "estpx", sizeof(double) * 4 * k * pl.px_parts, &ppx));
  RID_TRY(ws_get(c, "estax", sizeof(double) * 4 * m * pl.ax_parts, &pax));
  RID_TRY(ws_get(c, "estwall", sizeof(double) * 4 * m * (coll ? G : 1), &pwall));
  const int nparts_max = pl.z_blocks > pl.x0_blocks ? pl.z_blocks : pl.x0_blocks;
  RID_TRY(ws_get(c, "estnp", sizeof(double) * 2 * nparts_max, &pnp));
  RID_TRY(ws_get(c, "estnn", sizeof(double) * 2 * (G + 1), &pnn));
  RID_TRY(ws_get(c, "estval", sizeof(double), &pest));
  // bounds of the fixed-offset accumulation: [amax, xmax] for A x, [amax, ymax] for A^H y
  void* pmax;
  RID_TRY(ws_get(c, "estmax", sizeof(unsigned long long) * 4, &pmax));
  unsigned long long* bax = (unsigned long long*)pmax;  // {amax, xmax}
  unsigned long long* bz = bax + 2;                     // {amax, ymax}
  double2* B = (double2*)pB;
  double2 *x = (double2*)px, *z = (double2*)pz, *y = (double2*)py;
  double *u = (double*)pu, *nn = (double*)pnn;
  // B = A[:, J], replicated on every rank (owners contribute their columns, the rest are 0);
  // a pivot outside [0, n) raises the flag read after the final synchronisation (RID_EINVAL)
  void* pbad;
  RID_TRY(ws_get(c, "estbad", sizeof(int), &pbad));
  RID_CUDA(c, cudaMemsetAsync(pbad, 0, sizeof(int), c->stream));
  RID_CUDA(c, cudaMemsetAsync(B, 0, sizeof(double2) * m * k, c->stream));
  RID_CUDA(c, rid::gather_columns((const double2*)a.dev, lda, m, (const int64_t*)pJ, k, col0, n_loc,
                                  n, B, m, (int*)pbad, c->stream));
  if (coll) RID_TRY(c->comm->allreduce_sum(c, (double*)B, (size_t)(2 * m * k)));
  // reduce a dd scalar over ranks: local parts -> nn[2*rank], allgather, merge -> nn[2*G]
  auto scalar_allreduce = [&](const double* parts, int nparts) -> rid_status {
    double* slot = nn + 2 * (coll ? c->rank : 0);
    RID_CUDA(c, rid::est_merge_scalar(parts, nparts, slot, c->stream));
    if (coll) {
      RID_TRY(c->comm->allgather(c, nn, 2));
      RID_CUDA(c, rid::est_merge_scalar(nn, G, nn + 2 * G, c->stream));
    }
    return RID_OK;
  };
  const double* nn_final = nn + (coll ? 2 * G : 0);
  RID_CUDA(c, rid::est_x0(seed, col0, n_loc, x, (double*)pnp, pl, c->stream));
  RID_TRY(scalar_allreduce((const double*)pnp, pl.x0_blocks));
  RID_CUDA(c, rid::est_normalise(x, n_loc, nn_final, x, nullptr, bax + 1, c->stream));
  // amax (the fixed-offset bound) comes from the first iteration's A x pass (Dot2 there)
  RID_CUDA(c, cudaEventRecord(ev[1], c->stream));
  for (int it = 0; it < q; ++it) {
    // u = P x (replicated after the exchange)
    double* u_loc = u + (size_t)4 * k * (coll ? c->rank : 0);
    RID_CUDA(c, rid::est_px((const double2*)p.dev, ldp, k, n_loc, x, (double*)ppx, u_loc, pl, c->stream));
    if (coll) {
      RID_TRY(c->comm->allgather(c, u, (size_t)(4 * k)));
      RID_CUDA(c, rid::est_merge_vec(u, G, k, (double*)psb, c->stream));  // sb as scratch
      RID_CUDA(c, cudaMemcpyAsync(u, psb, sizeof(double) * 4 * k, cudaMemcpyDeviceToDevice, c->stream));
    }
    // y = A x - B u (replicated)
    RID_CUDA(c, rid::est_ax((const double2*)a.dev, lda, m, n_loc, x, bax, (double*)pax, pl, c->stream,
                            it == 0));
    if (pl.tma && it == 0)
      RID_CUDA(c, cudaMemcpyAsync(bz, bax, sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                                  c->stream));
    if (coll) {
      double* w_loc = (double*)pwall + (size_t)4 * m * c->rank;
      RID_CUDA(c, rid::est_merge_vec((const double*)pax, pl.ax_parts, m, w_loc, c->stream));
      RID_TRY(c->comm->allgather(c, (double*)pwall, (size_t)(4 * m)));
      RID_CUDA(c, rid::est_y((const double*)pwall, G, m, B, m, k, u, y, bz + 1, c->stream));
    } else {
      RID_CUDA(c, rid::est_y((const double*)pax, pl.ax_parts, m, B, m, k, u, y, bz + 1, c->stream));
    }
    // sb = B^H y ; z = A^H y - P^H sb ; x = z / ||z||
    RID_CUDA(c, rid::est_bhy(B, m, m, k, y, (double*)psb, c->stream));
    RID_CUDA(c, rid::est_z((const double2*)a.dev, lda, m, n_loc, y, (const double2*)p.dev, ldp, k,
                           (const double*)psb, z, bz, (double*)pnp, pl, c->stream));
    RID_TRY(scalar_allreduce((const double*)pnp, pl.z_blocks));
    RID_CUDA(c, rid::est_normalise(z, n_loc, nn_final, x, (double*)pest, bax + 1, c->stream));
  }
  RID_CUDA(c, cudaEventRecord(ev[2], c->stream));
  int bad = 0;
  RID_CUDA(c, cudaMemcpyAsync(est, pest, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  RID_CUDA(c, cudaMemcpyAsync(&bad, pbad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RID_CUDA(c, cudaStreamSynchronize(c->stream));
  if (bad) return fail(c, RID_EINVAL, "rid_error_estimate: a pivot index lies outside [0, n)");
  if (diag) {
    rid_diag d{};
    d.t_total = ev_ms(ev[0], ev[2]) * 1e-3;
    d.t_h2d = ev_ms(ev[0], ev[1]) * 1e-3;
    d.launches = 3 + 3 + q * (3 + 4 + (coll ? 2 : 1) + 1);
    *diag = d;
  }
  return RID_OK;
}

}  // extern "C"
