// api.cu — the C ABI of libprony (include/prony.h): synchronous validation, workspace
// planning, and stream-ordered launches of the kernels in project.cu / vandermonde_ls.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/prony.h"
#include "common.cuh"
#include "project.cuh"
#include "vandermonde_ls.cuh"
#include "dense.cuh"

using namespace prony;

// NVTX range over each compute entry point (SURVEY §5 tracing): named ranges on the host timeline of nsys /
// ncu --nvtx; without an attached tool the push / pop are a few nanoseconds
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

cudaError_t prony::ensure_smem_attr(const void* fn, int bytes) {
  struct Entry {
    int dev;
    const void* fn;
    int bytes;
  };
  static std::mutex mu;
  static std::vector<Entry> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (Entry& x : done)
    if (x.dev == dev && x.fn == fn) {
      if (x.bytes >= bytes) return cudaSuccess;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess) x.bytes = bytes;
      return e;
    }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back({dev, fn, bytes});
  return e;
}

namespace {

int sm_count_current() {
  constexpr int kMaxDev = 64;
  static int cached[kMaxDev] = {};  // SM count per device ordinal (0: not queried yet)
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (dev >= 0 && dev < kMaxDev && __atomic_load_n(&cached[dev], __ATOMIC_RELAXED) > 0) return cached[dev];
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev >= 0 && dev < kMaxDev) __atomic_store_n(&cached[dev], sms, __ATOMIC_RELAXED);
  return sms;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// d, n, m validation shared by every entry point. On success writes N and the box size.
int validate_dnm(int d, int n, int m, int64_t* N_out) {
  if (d < 1 || d > PRONY_MAX_D || n < 1 || m < 1) return PRONY_ERR_INVALID;
  if (m > PRONY_MAX_M) return PRONY_ERR_RANGE;
  int64_t N = 1, box = 1;
  for (int i = 0; i < d; ++i) {
    N *= (n + 1);
    box *= (2 * (int64_t)n + 2);
    if (box >= (int64_t(1) << 31)) return PRONY_ERR_RANGE;
  }
  if (m > N) return PRONY_ERR_RANGE;
  if (N * (int64_t)((m + 7) / 8 * 8) >= (int64_t(1) << 31)) return PRONY_ERR_RANGE;  // int32 offsets into V / Vsum
  *N_out = N;
  return PRONY_OK;
}

// rows of T_l covered by units [u0, u1) in the given order
void unit_rows(int d, int n, int64_t N, int64_t u0, int64_t u1, int order, ProjGeom* g) {
  if (order == PRONY_UNITS_SHARED) {
    g->shared = 1;
    g->e0 = (int)u0;
    g->e1 = (int)u1;
    return;
  }
  for (int l = 0; l < d; ++l) {
    int64_t kb, ke;
    if (order == PRONY_UNITS_L_MAJOR) {
      kb = std::min(std::max(u0 - l * N, (int64_t)0), N);
      ke = std::min(std::max(u1 - l * N, (int64_t)0), N);
    } else {  // u = k*d + l  ->  k in [ceil((u0-l)/d), ceil((u1-l)/d))
      auto cdiv = [](int64_t a, int64_t b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); };
      kb = std::min(std::max(cdiv(u0 - l, d), (int64_t)0), N);
      ke = std::min(std::max(cdiv(u1 - l, d), (int64_t)0), N);
    }
    g->kb[l] = (int)kb;
    g->rows[l] = (int)std::max<int64_t>(ke - kb, 0);
  }
}

size_t ws_project(int d, int n, int64_t N, int m, int sms) { return project_workspace_bytes(d, n, (int)N, m, sms); }
size_t ws_ls(int d, int n, int m, int sms) { return ls_workspace_bytes(d, n, m, sms); }
size_t ws_project_mu(int d, int n, int64_t N, int m, int sms) {
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  return align_up(ws_project(d, n, N, m, sms), 256) + align_up((size_t)box * sizeof(double2), 256) +
         align_up((size_t)d * m * m * sizeof(double2), 256);
}

// device copies used by prony_pencil_host, carved from the front of its workspace
struct HostLayout {
  size_t grid, U, V, sigma, z, S, G, b, c, t, status, inner, inner_ls, total;
};

HostLayout host_layout(int d, int n, int m, int64_t N, int sms) {
  HostLayout h{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes, 256);
    return o;
  };
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  h.grid = take(box * sizeof(double2));
  h.U = take(N * m * sizeof(double2));
  h.V = take(N * m * sizeof(double2));
  h.sigma = take(m * sizeof(double));
  h.z = take((size_t)m * d * sizeof(double2));
  h.S = take((size_t)d * m * m * sizeof(double2));
  h.G = take((size_t)m * m * sizeof(double2));
  h.b = take(m * sizeof(double2));
  h.c = take(m * sizeof(double2));
  h.t = take((size_t)m * d * sizeof(double));
  h.status = take(sizeof(int32_t));
  h.inner = off;  // projection and LS run concurrently: separate scratch
  off += align_up(ws_project(d, n, N, m, sms), 256);
  h.inner_ls = off;
  off += ws_ls(d, n, m, sms);
  h.total = off;
  return h;
}

}  // namespace

extern "C" {

int prony_abi_version(void) { return PRONY_ABI_VERSION; }

const char* prony_status_string(int status) {
  switch (status) {
    case PRONY_OK: return "ok";
    case PRONY_ERR_INVALID: return "invalid argument (null/misaligned pointer, d/n/m out of range, bad order)";
    case PRONY_ERR_RANGE: return "size out of range ((2n+2)^d >= 2^31, m > max, m > N, range outside limits)";
    case PRONY_ERR_SINGULAR: return "numerically singular (G not Hermitian positive definite)";
    case PRONY_ERR_RANK: return "detected rank below m";
    case PRONY_ERR_NOT_CONVERGED: return "iteration did not converge";
    case PRONY_ERR_CUDA: return "CUDA error";
    case PRONY_ERR_UNIMPLEMENTED: return "not implemented in this build";
    case PRONY_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int prony_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PRONY_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return PRONY_ERR_CUDA;
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return PRONY_OK;
}

int prony_workspace_size(int kind, int d, int n, int m, size_t* bytes) {
  if (!bytes) return PRONY_ERR_INVALID;
  int64_t N = 0;
  if (kind == PRONY_WS_DIAG) {  // the diagonalization does not depend on n: only d and m are checked
    if (d < 1 || d > PRONY_MAX_D || m < 1) return PRONY_ERR_INVALID;
    if (m > PRONY_MAX_M) return PRONY_ERR_RANGE;
    *bytes = diag_workspace_bytes(d, m);
    return PRONY_OK;
  }
  if (kind == PRONY_WS_LANCZOS) {
    const int rc = validate_dnm(d, n, 1, &N);
    if (rc) return rc;
    if (m < 1 || m > kLanczosMaxRank || m > N) return PRONY_ERR_RANGE;
    *bytes = lanczos_workspace_bytes(d, n, (int)N, m);
    return PRONY_OK;
  }
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  switch (kind) {
    case PRONY_WS_PROJECT: *bytes = ws_project(d, n, N, m, sms); return PRONY_OK;
    case PRONY_WS_LS: *bytes = ws_ls(d, n, m, sms); return PRONY_OK;
    case PRONY_WS_PENCIL_HOST: *bytes = host_layout(d, n, m, N, sms).total; return PRONY_OK;
    case PRONY_WS_BUILD:
      *bytes = std::max(svd_workspace_bytes(d, n, (int)N, m), ws_project(d, n, N, m, sms));
      return PRONY_OK;
    case PRONY_WS_PROJECT_MU: *bytes = ws_project_mu(d, n, N, m, sms); return PRONY_OK;
    case PRONY_WS_PENCIL: *bytes = align_up(ws_project(d, n, N, m, sms), 256) + ws_ls(d, n, m, sms); return PRONY_OK;
    case PRONY_WS_APPLY: *bytes = apply_workspace_bytes(d, n, (int)N); return PRONY_OK;
    default: return PRONY_ERR_INVALID;
  }
}

int prony_project(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                  const double* sigma, int64_t unit_begin, int64_t unit_end, int unit_order, prony_c128* S,
                  void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream) {
  return prony_project_ex(d, n, m, grid, U, V, sigma, unit_begin, unit_end, unit_order, S, workspace,
                          workspace_bytes, dev_status, stream, nullptr);
}

int prony_project_ex(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                     const double* sigma, int64_t unit_begin, int64_t unit_end, int unit_order, prony_c128* S,
                     void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream,
                     prony_exec_info* info) {
  NvtxRange nvtx_("prony_project_ex");
  int64_t N = 0;
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  if (!grid || !U || !V || !sigma || !S || !workspace) return PRONY_ERR_INVALID;
  if (!aligned16(grid) || !aligned16(U) || !aligned16(V) || !aligned16(S) || ((uintptr_t)sigma & 7u) ||
      ((uintptr_t)workspace & 255u))
    return PRONY_ERR_INVALID;
  if (unit_order != PRONY_UNITS_L_MAJOR && unit_order != PRONY_UNITS_ROW_MAJOR && unit_order != PRONY_UNITS_SHARED)
    return PRONY_ERR_INVALID;
  const int64_t units = unit_order == PRONY_UNITS_SHARED ? ext_rows(d, n) : (int64_t)d * N;
  if (unit_begin < 0 || unit_end < unit_begin || unit_end > units) return PRONY_ERR_RANGE;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  if (workspace_bytes < ws_project(d, n, N, m, sms)) return PRONY_ERR_WORKSPACE;
  ProjGeom g{};
  g.d = d;
  g.n = n;
  g.m = m;
  g.N = (int)N;
  unit_rows(d, n, N, unit_begin, unit_end, unit_order, &g);
  ProjPlan pl{};
  project_plan(g, sms, &pl);
  return project_launch(g, pl, (const double2*)grid, (const double2*)U, (const double2*)V, sigma, (double2*)S,
                        workspace, sms, (cudaStream_t)stream, info,
                        info ? (cudaEvent_t)info->ev_wait_u : nullptr, 1, dev_status);
}

int prony_vandermonde_ls(int d, int n, int m, const prony_c128* z, const prony_c128* grid, int64_t col_begin,
                         int64_t col_end, prony_c128* A, prony_c128* G, prony_c128* b, prony_c128* c, double* t,
                         void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream) {
  return prony_vandermonde_ls_ex(d, n, m, z, grid, col_begin, col_end, A, G, b, c, t, workspace, workspace_bytes,
                                 dev_status, stream, nullptr);
}

int prony_vandermonde_ls_ex(int d, int n, int m, const prony_c128* z, const prony_c128* grid, int64_t col_begin,
                            int64_t col_end, prony_c128* A, prony_c128* G, prony_c128* b, prony_c128* c, double* t,
                            void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream,
                            prony_exec_info* info) {
  NvtxRange nvtx_("prony_vandermonde_ls_ex");
  int64_t N = 0;
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  if (!z || !grid || !G || !b || !workspace) return PRONY_ERR_INVALID;
  if (!aligned16(z) || !aligned16(grid) || !aligned16(G) || !aligned16(b) || (A && !aligned16(A)) ||
      (c && !aligned16(c)) || (t && ((uintptr_t)t & 7u)) || ((uintptr_t)workspace & 255u))
    return PRONY_ERR_INVALID;
  if (col_begin < 0 || col_end < col_begin || col_end > N) return PRONY_ERR_RANGE;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  if (workspace_bytes < ws_ls(d, n, m, sms)) return PRONY_ERR_WORKSPACE;
  return ls_launch(d, n, m, (int)N, (const double2*)z, (const double2*)grid, col_begin, col_end, (double2*)A,
                   (double2*)G, (double2*)b, (double2*)c, t, workspace, dev_status, sms, (cudaStream_t)stream, info);
}

int prony_ls_solve(int d, int m, const prony_c128* G, const prony_c128* b, const prony_c128* z, prony_c128* c,
                   double* t, void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream) {
  NvtxRange nvtx_("prony_ls_solve");
  if (d < 1 || d > PRONY_MAX_D || m < 1) return PRONY_ERR_INVALID;
  if (m > PRONY_MAX_M) return PRONY_ERR_RANGE;
  (void)workspace_bytes;  // the solve keeps its factor in shared memory; no scratch is needed
  if (!G || !b || !z || !c) return PRONY_ERR_INVALID;
  if (!aligned16(G) || !aligned16(b) || !aligned16(z) || !aligned16(c) || (t && ((uintptr_t)t & 7u)))
    return PRONY_ERR_INVALID;
  return ls_solve_launch(d, m, (const double2*)G, (const double2*)b, (const double2*)z, (double2*)c, t, workspace,
                         dev_status, (cudaStream_t)stream);
}

int prony_project_mu(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                     const double* sigma, const prony_c128* mu, prony_c128* C, void* workspace, size_t workspace_bytes,
                     int32_t* dev_status, prony_stream_t stream) {
  NvtxRange nvtx_("prony_project_mu");
  int64_t N = 0;
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  if (!grid || !U || !V || !sigma || !mu || !C || !workspace) return PRONY_ERR_INVALID;
  if (!aligned16(grid) || !aligned16(U) || !aligned16(V) || !aligned16(mu) || !aligned16(C) || ((uintptr_t)sigma & 7u) ||
      ((uintptr_t)workspace & 255u))
    return PRONY_ERR_INVALID;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  if (workspace_bytes < ws_project_mu(d, n, N, m, sms)) return PRONY_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  const size_t off_g = align_up(ws_project(d, n, N, m, sms), 256);
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  const size_t off_s = off_g + align_up((size_t)box * sizeof(double2), 256);
  double2* gmu = (double2*)(w + off_g);
  double2* Sd = (double2*)(w + off_s);
  k_combine_grid<<<2 * sms, 256, 0, st>>>(d, n, box, (const double2*)grid, (const double2*)mu, gmu);
  ProjGeom g{};
  g.d = d;
  g.n = n;
  g.m = m;
  g.N = (int)N;
  g.kb[0] = 0;
  g.rows[0] = (int)N;  // one segment: the l = 0 operator on the combined grid
  ProjPlan pl{};
  project_plan(g, sms, &pl);
  rc = project_launch(g, pl, gmu, (const double2*)U, (const double2*)V, sigma, Sd, w, sms, st, nullptr, nullptr, 0,
                      dev_status);
  if (rc) return rc;
  if (cudaMemcpyAsync(C, Sd, (size_t)m * m * sizeof(double2), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return PRONY_ERR_CUDA;
  return PRONY_OK;
}

int prony_toeplitz_apply(int d, int n, const prony_c128* grid, int ell, int conj, const prony_c128* X, int ldx, int r,
                         prony_c128* Y, int ldy, void* workspace, size_t workspace_bytes, prony_stream_t stream) {
  NvtxRange nvtx_("prony_toeplitz_apply");
  int64_t N = 0;
  int rc = validate_dnm(d, n, 1, &N);
  if (rc) return rc;
  if (ell < 0 || ell > d || (conj && ell != 0) || r < 1 || ldx < r || ldy < r) return PRONY_ERR_INVALID;
  if (!grid || !X || !Y || !workspace) return PRONY_ERR_INVALID;
  if (!aligned16(grid) || !aligned16(X) || !aligned16(Y) || ((uintptr_t)workspace & 255u)) return PRONY_ERR_INVALID;
  if (N * (int64_t)std::max(ldx, ldy) >= (int64_t(1) << 31)) return PRONY_ERR_RANGE;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  if (workspace_bytes < apply_workspace_bytes(d, n, (int)N)) return PRONY_ERR_WORKSPACE;
  return toeplitz_apply_launch(d, n, (int)N, (const double2*)grid, ell, conj, (const double2*)X, ldx, r, (double2*)Y,
                               ldy, workspace, sms, (cudaStream_t)stream);
}

}  // extern "C"

namespace {

// Rows of U that the SHARED units [e0, e1) pair with (over all l): k = k' - e_l for the k' of the slab
// with k in I_n. For fixed l that row index is increasing in k', so the range is bounded by the first
// and the last valid unit of the slab for each l.
void shared_u_rows(int d, int n, int64_t e0, int64_t e1, int64_t* lo, int64_t* hi) {
  const int Le = n + 2;
  auto krow = [&](int64_t e, int l) -> int64_t {  // -1 if k' - e_l is outside I_n
    int c[PRONY_MAX_D];
    for (int i = d - 1; i >= 0; --i) {
      c[i] = (int)(e % Le);
      e /= Le;
    }
    c[l] -= 1;
    int64_t k = 0;
    for (int i = 0; i < d; ++i) {
      if (c[i] < 0 || c[i] > n) return -1;
      k = k * (n + 1) + c[i];
    }
    return k;
  };
  *lo = INT64_MAX;
  *hi = -1;
  for (int l = 0; l < d; ++l) {
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t k = krow(e, l);
      if (k >= 0) {
        *lo = std::min(*lo, k);
        break;
      }
    }
    for (int64_t e = e1 - 1; e >= e0; --e) {
      const int64_t k = krow(e, l);
      if (k >= 0) {
        *hi = std::max(*hi, k + 1);
        break;
      }
    }
  }
  if (*hi < 0) *lo = *hi = 0;
}

}  // namespace

// Streams and events of the host-input pencil (prony_pencil_host*): created once by
// prony_host_context_create and reused by every call that passes the context, or created and destroyed by
// a call that passes none.
struct prony_host_context_s {
  int device = -1;
  cudaStream_t s2 = nullptr, s3 = nullptr, s4 = nullptr;
  cudaStream_t sl[kSplitStreams] = {};     // launch streams of the later split-K chunk groups
  cudaEvent_t ev[8] = {};  // in, grid, v0, u, done, split a, split b, v rest
  cudaEvent_t ev_chunk[kMaxChunkEv] = {};  // V rows of split-K chunk c >= 1 copied
  cudaEvent_t ev_join[kSplitStreams] = {};
};

namespace {

void host_ctx_release(prony_host_context_s* c) {
  for (cudaEvent_t& e : c->ev)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  for (cudaEvent_t* arr : {c->ev_chunk, c->ev_join})
    for (int i = 0; i < (arr == c->ev_chunk ? kMaxChunkEv : kSplitStreams); ++i)
      if (arr[i]) {
        cudaEventDestroy(arr[i]);
        arr[i] = nullptr;
      }
  for (cudaStream_t* s : {&c->s2, &c->s3, &c->s4, &c->sl[0], &c->sl[1], &c->sl[2]})
    if (*s) {
      cudaStreamDestroy(*s);
      *s = nullptr;
    }
}

int host_ctx_init(prony_host_context_s* c) {
  if (cudaGetDevice(&c->device) != cudaSuccess) return PRONY_ERR_CUDA;
  bool good = cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->s3, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->s4, cudaStreamNonBlocking) == cudaSuccess;
  for (int i = 0; i < kSplitStreams && good; ++i)
    good = cudaStreamCreateWithFlags(&c->sl[i], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; i < 8 && good; ++i) good = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; i < kMaxChunkEv && good; ++i)
    good = cudaEventCreateWithFlags(&c->ev_chunk[i], cudaEventDisableTiming) == cudaSuccess;
  if (!good) {
    host_ctx_release(c);
    return PRONY_ERR_CUDA;
  }
  return PRONY_OK;
}

// PRONY_HOST_TIMELINE=1 (diagnostic): timing events at the stages of host_pencil, printed to stderr by
// prony_pencil_host_ctx after its synchronize (ms from the call's start on `st`)
struct HostTimeline {
  bool on = false;
  cudaEvent_t e[10] = {};
  const char* name[10] = {"grid+V0+sigma", "-", "proj0_begin", "proj0_end", "Vrest", "proj_reduced", "U", "LS_end",
                          "end", "start"};
};
HostTimeline& host_timeline() {
  static HostTimeline t = [] {
    HostTimeline x;
    const char* e = getenv("PRONY_HOST_TIMELINE");
    x.on = e && atoi(e) > 0;
    if (x.on)
      for (auto& ev : x.e) cudaEventCreate(&ev);
    return x;
  }();
  return t;
}

// Host-input pencil on the device (prony_pencil_host / prony_pencil_host_part). The link carries, in order:
// on `st` the grid, the V rows of the narrow split-K chunk 0 (project_plan_lead) and sigma -> k_prep ->
// chunk 0 of the projection; on the copy stream `s2` the V rows of chunk 1, 2, ... (an event after each);
// on `s4` the U rows after all of V (first needed by k_reduce); `s3` carries z and, once the prep kernels are
// done, the LS step. The later chunks of the projection run in groups on the context's launch streams, each
// as soon as ITS rows are in, so only chunk 0's rows (about 1/24 of V) are copied before the first DMMA and each
// later chunk's copy hides behind the chunks before it. On return `st` is ordered after everything. The streams /
// events come from `ctx` (a caller's context) or are created for this call.
int host_pencil(int d, int n, int m, int64_t N, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                const double* sigma, const prony_c128* z, int64_t e0, int64_t e1, int64_t c0, int64_t c1, bool solve,
                double2* S_dev, double2* G_dev, double2* b_dev, double2* c_dev, double* t_dev, int32_t* dst,
                char* w, const HostLayout& h, int sms, cudaStream_t st, prony_host_context_s* ctx) {
  int64_t box = 1;
  for (int i = 0; i < d; ++i) box *= (2 * (int64_t)n + 2);
  ProjGeom g{};
  g.d = d;
  g.n = n;
  g.m = m;
  g.N = (int)N;
  unit_rows(d, n, N, e0, e1, PRONY_UNITS_SHARED, &g);
  ProjPlan pl{};
  project_plan(g, sms, &pl);
  project_plan_lead(g, &pl);  // a narrow chunk 0: only its V rows are copied before the first DMMA
  const bool split = pl.KC > 1;
  const int64_t v0 = split ? std::min<int64_t>(pl.chunk0_w, N) : N;
  int64_t ulo = 0, uhi = N;
  if (e0 != 0 || e1 != ext_rows(d, n)) shared_u_rows(d, n, e0, e1, &ulo, &uhi);
  prony_host_context_s local;
  const bool own = ctx == nullptr;
  if (own) {
    if (host_ctx_init(&local) != PRONY_OK) return PRONY_ERR_CUDA;
    ctx = &local;
  } else {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return PRONY_ERR_CUDA;
    if (dev != ctx->device) return PRONY_ERR_INVALID;
  }
  cudaStream_t s2 = ctx->s2, s3 = ctx->s3, s4 = ctx->s4;
  cudaEvent_t* ev = ctx->ev;
  cudaEvent_t ev_prep = ev[0], ev_grid = ev[1], ev_v0 = ev[2], ev_u = ev[3], ev_done = ev[4], ev_vrest = ev[7];
  auto ok = [](cudaError_t e) { return e == cudaSuccess; };
  const size_t vrow = (size_t)m * sizeof(double2);
  HostTimeline& tl = host_timeline();
  if (tl.on) cudaEventRecord(tl.e[9], st);
  bool good = ok(cudaMemcpyAsync(w + h.grid, grid, box * sizeof(double2), cudaMemcpyHostToDevice, st)) &&
              ok(cudaEventRecord(ev_grid, st)) &&
              ok(cudaMemcpyAsync(w + h.V, V, v0 * vrow, cudaMemcpyHostToDevice, st)) &&
              ok(cudaMemcpyAsync(w + h.sigma, sigma, m * sizeof(double), cudaMemcpyHostToDevice, st)) &&
              ok(cudaEventRecord(ev_v0, st)) && ok(cudaStreamWaitEvent(s2, ev_v0, 0));
  for (int c = 1; good && split && c < pl.KC; ++c) {  // chunk c's V rows, then its event
    const int64_t r0 = pl.chunk0_w + (int64_t)(c - 1) * pl.chunk_w, r1 = std::min<int64_t>(r0 + pl.chunk_w, N);
    good = ok(cudaMemcpyAsync(w + h.V + r0 * vrow, (const char*)V + r0 * vrow, (r1 - r0) * vrow,
                              cudaMemcpyHostToDevice, s2)) &&
           ok(cudaEventRecord(ctx->ev_chunk[std::min(c - 1, kMaxChunkEv - 1)], s2));
  }
  good = good && ok(cudaEventRecord(ev_vrest, s2)) && ok(cudaStreamWaitEvent(s4, ev_vrest, 0)) &&
         (uhi <= ulo || ok(cudaMemcpyAsync(w + h.U + ulo * vrow, (const char*)U + ulo * vrow, (uhi - ulo) * vrow,
                                           cudaMemcpyHostToDevice, s4))) &&
         ok(cudaEventRecord(ev_u, s4)) && ok(cudaStreamWaitEvent(s3, ev_grid, 0)) &&
         ok(cudaMemcpyAsync(w + h.z, z, (size_t)m * d * sizeof(double2), cudaMemcpyHostToDevice, s3));
  int rc = good ? PRONY_OK : PRONY_ERR_CUDA;
  prony_exec_info tinfo{};
  if (tl.on) {
    cudaEventRecord(tl.e[0], st);
    cudaEventRecord(tl.e[4], s2);
    cudaEventRecord(tl.e[6], s4);
    tinfo.ev_main_begin = tl.e[2];
    tinfo.ev_main_end = tl.e[3];
  }
  if (rc == PRONY_OK) {
    ProjSplit sp{{ctx->sl[0], ctx->sl[1], ctx->sl[2]}, ev[5], {ctx->ev_join[0], ctx->ev_join[1], ctx->ev_join[2]},
                 ctx->ev_chunk};
    rc = project_launch(g, pl, (const double2*)(w + h.grid), (const double2*)(w + h.U), (const double2*)(w + h.V),
                        (const double*)(w + h.sigma), S_dev, w + h.inner, sms, st, tl.on ? &tinfo : nullptr, ev_u, 1,
                        dst, split ? &sp : nullptr, ev_prep);
    if (tl.on) cudaEventRecord(tl.e[5], st);
  }
  // the LS step starts once the prep kernels are done and chunk 0 is enqueued (as in prony_pencil): its CTAs
  // then fill the SMs the projection leaves idle instead of delaying its first wave
  if (rc == PRONY_OK && !ok(cudaStreamWaitEvent(s3, ev_prep, 0))) rc = PRONY_ERR_CUDA;
  if (rc == PRONY_OK)
    rc = ls_launch(d, n, m, (int)N, (const double2*)(w + h.z), (const double2*)(w + h.grid), c0, c1, nullptr, G_dev,
                   b_dev, solve ? c_dev : nullptr, solve ? t_dev : nullptr, w + h.inner_ls, dst, sms, s3, nullptr);
  if (tl.on) cudaEventRecord(tl.e[7], s3);
  // `st` ends after everything the call enqueued on s2..s4 and the launch streams (s2 through s4's U copy, the launch
  // streams through project_launch's joins; also when the projection had nothing to do and never waited on them): the
  // host buffers may be released once `st` is synchronized, and a context's streams are idle for the next call once
  // `st` gets here
  if (rc == PRONY_OK && !(ok(cudaEventRecord(ev_done, s3)) && ok(cudaStreamWaitEvent(st, ev_done, 0)) &&
                          ok(cudaEventRecord(ev_u, s4)) && ok(cudaStreamWaitEvent(st, ev_u, 0))))
    rc = PRONY_ERR_CUDA;
  if (rc != PRONY_OK)
    for (cudaStream_t s : {s2, s3, s4, ctx->sl[0], ctx->sl[1], ctx->sl[2]}) cudaStreamSynchronize(s);
  if (own) host_ctx_release(&local);
  return rc;
}

}  // namespace

extern "C" {

int prony_host_context_create(prony_host_context* out) {
  if (!out) return PRONY_ERR_INVALID;
  *out = nullptr;
  prony_host_context_s* c = new (std::nothrow) prony_host_context_s();
  if (!c) return PRONY_ERR_CUDA;
  const int rc = host_ctx_init(c);
  if (rc != PRONY_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return PRONY_OK;
}

int prony_host_context_destroy(prony_host_context ctx) {
  if (!ctx) return PRONY_ERR_INVALID;
  for (cudaStream_t s : {ctx->s2, ctx->s3, ctx->s4, ctx->sl[0], ctx->sl[1], ctx->sl[2]})
    if (s) cudaStreamSynchronize(s);
  host_ctx_release(ctx);
  delete ctx;
  return PRONY_OK;
}

int prony_pencil(prony_host_context ctx, int d, int n, int m, const prony_c128* grid, const prony_c128* U,
                 const prony_c128* V, const double* sigma, const prony_c128* z, prony_c128* S, prony_c128* G,
                 prony_c128* b, prony_c128* c, double* t, void* workspace, size_t workspace_bytes,
                 int32_t* dev_status, prony_stream_t stream, prony_exec_info* info_project,
                 prony_exec_info* info_ls) {
  NvtxRange nvtx_("prony_pencil");
  int64_t N = 0;
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  if (!grid || !U || !V || !sigma || !z || !S || !G || !b || !workspace) return PRONY_ERR_INVALID;
  if (!aligned16(grid) || !aligned16(U) || !aligned16(V) || !aligned16(z) || !aligned16(S) || !aligned16(G) ||
      !aligned16(b) || (c && !aligned16(c)) || (t && ((uintptr_t)t & 7u)) || ((uintptr_t)sigma & 7u) ||
      ((uintptr_t)workspace & 255u))
    return PRONY_ERR_INVALID;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  const size_t off_ls = align_up(ws_project(d, n, N, m, sms), 256);
  if (workspace_bytes < off_ls + ws_ls(d, n, m, sms)) return PRONY_ERR_WORKSPACE;
  prony_host_context_s local;
  const bool own = ctx == nullptr;
  if (own) {
    if (host_ctx_init(&local) != PRONY_OK) return PRONY_ERR_CUDA;
    ctx = &local;
  } else {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return PRONY_ERR_CUDA;
    if (dev != ctx->device) return PRONY_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream, side = ctx->s3;
  cudaEvent_t ev_in = ctx->ev[0], ev_done = ctx->ev[4];
  ProjGeom g{};
  g.d = d;
  g.n = n;
  g.m = m;
  g.N = (int)N;
  unit_rows(d, n, N, 0, ext_rows(d, n), PRONY_UNITS_SHARED, &g);
  ProjPlan pl{};
  project_plan(g, sms, &pl);
  char* w = (char*)workspace;
  // the LS side stream starts once the prep kernels are done and k_project is enqueued (ev_in, recorded by
  // project_launch): were it released at the call's start, back-to-back calls would let k_vls (one CTA per SM)
  // take the SMs ahead of k_project's first wave (measured: k_project delayed 0.1 ms per pencil at cfg4); this
  // way k_project is served first and the LS CTAs fill the SMs its last wave leaves idle
  rc = project_launch(g, pl, (const double2*)grid, (const double2*)U, (const double2*)V, sigma, (double2*)S, w,
                      sms, st, info_project, nullptr, 1, dev_status, nullptr, ev_in, /*reset_status=*/true);
  if (rc == PRONY_OK && cudaStreamWaitEvent(side, ev_in, 0) != cudaSuccess) rc = PRONY_ERR_CUDA;
  if (rc == PRONY_OK)
    rc = ls_launch(d, n, m, (int)N, (const double2*)z, (const double2*)grid, 0, N, nullptr, (double2*)G, (double2*)b,
                   (double2*)c, t, w + off_ls, dev_status, sms, side, info_ls);
  if (rc == PRONY_OK && !(cudaEventRecord(ev_done, side) == cudaSuccess &&
                          cudaStreamWaitEvent(st, ev_done, 0) == cudaSuccess))
    rc = PRONY_ERR_CUDA;
  if (rc != PRONY_OK) cudaStreamSynchronize(side);
  if (own) host_ctx_release(&local);
  return rc;
}

int prony_pencil_host(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                      const double* sigma, const prony_c128* z, prony_c128* S, prony_c128* G, prony_c128* b,
                      prony_c128* c, double* t, void* workspace, size_t workspace_bytes, int32_t* status_out,
                      prony_stream_t stream) {
  return prony_pencil_host_ctx(nullptr, d, n, m, grid, U, V, sigma, z, S, G, b, c, t, workspace, workspace_bytes,
                               status_out, stream);
}

int prony_pencil_host_ctx(prony_host_context ctx, int d, int n, int m, const prony_c128* grid, const prony_c128* U,
                          const prony_c128* V, const double* sigma, const prony_c128* z, prony_c128* S, prony_c128* G,
                          prony_c128* b, prony_c128* c, double* t, void* workspace, size_t workspace_bytes,
                          int32_t* status_out, prony_stream_t stream) {
  NvtxRange nvtx_("prony_pencil_host_ctx");
  int64_t N = 0;
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  if (!grid || !U || !V || !sigma || !z || !workspace) return PRONY_ERR_INVALID;
  if ((uintptr_t)workspace & 255u) return PRONY_ERR_INVALID;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  const HostLayout h = host_layout(d, n, m, N, sms);
  if (workspace_bytes < h.total) return PRONY_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  int32_t* dst = (int32_t*)(w + h.status);
  if (cudaMemsetAsync(dst, 0, sizeof(int32_t), st) != cudaSuccess) return PRONY_ERR_CUDA;
  rc = host_pencil(d, n, m, N, grid, U, V, sigma, z, 0, ext_rows(d, n), 0, N, true, (double2*)(w + h.S),
                   (double2*)(w + h.G), (double2*)(w + h.b), (double2*)(w + h.c), (double*)(w + h.t), dst, w, h, sms,
                   st, ctx);
  if (rc != PRONY_OK) return rc;
  auto d2h = [&](void* dstp, size_t off, size_t bytes) {
    return dstp == nullptr || cudaMemcpyAsync(dstp, w + off, bytes, cudaMemcpyDeviceToHost, st) == cudaSuccess;
  };
  const bool good = d2h(S, h.S, (size_t)d * m * m * sizeof(double2)) && d2h(G, h.G, (size_t)m * m * sizeof(double2)) &&
                    d2h(b, h.b, m * sizeof(double2)) && d2h(c, h.c, m * sizeof(double2)) &&
                    d2h(t, h.t, (size_t)m * d * sizeof(double)) && d2h(status_out, h.status, sizeof(int32_t));
  HostTimeline& tl = host_timeline();
  if (tl.on) cudaEventRecord(tl.e[8], st);
  const bool synced = good && cudaStreamSynchronize(st) == cudaSuccess;
  if (synced && tl.on) {
    fprintf(stderr, "PRONY_HOST_TIMELINE");
    for (int i = 0; i < 9; ++i) {
      float ms = -1.0f;
      if (i != 1) cudaEventElapsedTime(&ms, tl.e[9], tl.e[i]);  // e[1] unused (the prep event is the context's)
      if (i != 1) fprintf(stderr, " %s=%.3f", tl.name[i], ms);
    }
    fprintf(stderr, "\n");
    (void)cudaGetLastError();
  }
  return synced ? PRONY_OK : PRONY_ERR_CUDA;
}

int prony_pencil_host_part(int d, int n, int m, const prony_c128* grid, const prony_c128* U, const prony_c128* V,
                           const double* sigma, const prony_c128* z, int64_t unit_begin, int64_t unit_end,
                           int64_t col_begin, int64_t col_end, prony_c128* S, prony_c128* G, prony_c128* b,
                           void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream) {
  return prony_pencil_host_part_ctx(nullptr, d, n, m, grid, U, V, sigma, z, unit_begin, unit_end, col_begin, col_end,
                                    S, G, b, workspace, workspace_bytes, dev_status, stream);
}

int prony_pencil_host_part_ctx(prony_host_context ctx, int d, int n, int m, const prony_c128* grid,
                               const prony_c128* U, const prony_c128* V, const double* sigma, const prony_c128* z,
                               int64_t unit_begin, int64_t unit_end, int64_t col_begin, int64_t col_end, prony_c128* S,
                               prony_c128* G, prony_c128* b, void* workspace, size_t workspace_bytes,
                               int32_t* dev_status, prony_stream_t stream) {
  NvtxRange nvtx_("prony_pencil_host_part_ctx");
  int64_t N = 0;
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  if (!grid || !U || !V || !sigma || !z || !S || !G || !b || !workspace) return PRONY_ERR_INVALID;
  if (!aligned16(S) || !aligned16(G) || !aligned16(b) || ((uintptr_t)workspace & 255u)) return PRONY_ERR_INVALID;
  if (unit_begin < 0 || unit_end < unit_begin || unit_end > ext_rows(d, n)) return PRONY_ERR_RANGE;
  if (col_begin < 0 || col_end < col_begin || col_end > N) return PRONY_ERR_RANGE;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  const HostLayout h = host_layout(d, n, m, N, sms);
  if (workspace_bytes < h.total) return PRONY_ERR_WORKSPACE;
  return host_pencil(d, n, m, N, grid, U, V, sigma, z, unit_begin, unit_end, col_begin, col_end, false, (double2*)S,
                     (double2*)G, (double2*)b, nullptr, nullptr, dev_status, (char*)workspace, h, sms,
                     (cudaStream_t)stream, ctx);
}

int prony_build_pencil(int d, int n, int m, const prony_c128* grid, uint64_t seed, double tol, int max_iter,
                       prony_c128* S, prony_c128* U, prony_c128* V, double* sigma, int32_t* rank_out,
                       double* resid_out, void* workspace, size_t workspace_bytes, int32_t* dev_status,
                       prony_stream_t stream) {
  NvtxRange nvtx_("prony_build_pencil");
  int64_t N = 0;
  int rc = validate_dnm(d, n, m, &N);
  if (rc) return rc;
  if (!grid || !S || !U || !V || !sigma || !rank_out || !workspace || max_iter < 1 || !(tol >= 0.0))
    return PRONY_ERR_INVALID;
  if (!aligned16(grid) || !aligned16(S) || !aligned16(U) || !aligned16(V) || ((uintptr_t)sigma & 7u) ||
      ((uintptr_t)workspace & 255u))
    return PRONY_ERR_INVALID;
  if (2 * m > 256) return PRONY_ERR_RANGE;  // starting block 2m columns: Jacobi pair table limit
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  const size_t need = std::max(svd_workspace_bytes(d, n, (int)N, m), ws_project(d, n, N, m, sms));
  if (workspace_bytes < need) return PRONY_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  int rank = 0, iters = 0;
  double resid = -1.0;
  const int src = block_power_svd(d, n, (int)N, (const double2*)grid, m, tol, max_iter, seed, (double2*)U,
                                  (double2*)V, sigma, &rank, &iters, &resid, workspace, sms, st);
  *rank_out = rank;
  if (resid_out) *resid_out = resid;
  if (src != PRONY_OK && src != PRONY_ERR_NOT_CONVERGED) return src;
  rc = prony_project(d, n, m, grid, U, V, sigma, 0, ext_rows(d, n), PRONY_UNITS_SHARED, S, workspace,
                     workspace_bytes, dev_status, stream);
  if (rc) return rc;
  if (cudaStreamSynchronize(st) != cudaSuccess) return PRONY_ERR_CUDA;
  return src;
}

int prony_lanczos_svd(int d, int n, const prony_c128* grid, int max_rank, double tol, uint64_t seed, int ldo,
                      prony_c128* U, prony_c128* V, double* sigma, int32_t* rank_out, int32_t* steps_out,
                      void* workspace, size_t workspace_bytes, prony_stream_t stream) {
  NvtxRange nvtx_("prony_lanczos_svd");
  int64_t N = 0;
  int rc = validate_dnm(d, n, 1, &N);
  if (rc) return rc;
  if (!grid || !U || !V || !sigma || !rank_out || !workspace || !(tol >= 0.0)) return PRONY_ERR_INVALID;
  if (max_rank < 1 || ldo < 1 || ldo > max_rank) return PRONY_ERR_INVALID;
  if (max_rank > kLanczosMaxRank || max_rank > N) return PRONY_ERR_RANGE;
  if (!aligned16(grid) || !aligned16(U) || !aligned16(V) || ((uintptr_t)sigma & 7u) || ((uintptr_t)workspace & 255u))
    return PRONY_ERR_INVALID;
  if (workspace_bytes < lanczos_workspace_bytes(d, n, (int)N, max_rank)) return PRONY_ERR_WORKSPACE;
  const int sms = sm_count_current();
  if (sms <= 0) return PRONY_ERR_CUDA;
  int rank = 0, steps = 0;
  rc = lanczos_svd(d, n, (int)N, (const double2*)grid, max_rank, tol, seed, (double2*)U, (double2*)V, sigma, ldo,
                   &rank, &steps, workspace, sms, (cudaStream_t)stream);
  *rank_out = rank;
  if (steps_out) *steps_out = steps;
  return rc;
}

int prony_diagonalize(int d, int m, const prony_c128* S, const prony_c128* mu, prony_c128* z, double* t, prony_c128* W,
                      void* workspace, size_t workspace_bytes, int32_t* dev_status, prony_stream_t stream) {
  NvtxRange nvtx_("prony_diagonalize");
  if (d < 1 || d > PRONY_MAX_D || m < 1) return PRONY_ERR_INVALID;
  if (m > PRONY_MAX_M) return PRONY_ERR_RANGE;
  if (!S || !mu || !z || !W || !workspace) return PRONY_ERR_INVALID;
  if (!aligned16(S) || !aligned16(mu) || !aligned16(z) || !aligned16(W) || (t && ((uintptr_t)t & 7u)) ||
      ((uintptr_t)workspace & 255u))
    return PRONY_ERR_INVALID;
  if (workspace_bytes < diag_workspace_bytes(d, m)) return PRONY_ERR_WORKSPACE;
  return diagonalize_launch(d, m, (const double2*)S, (const double2*)mu, (double2*)z, t, (double2*)W, workspace,
                            dev_status, (cudaStream_t)stream);
}

}  // extern "C"
