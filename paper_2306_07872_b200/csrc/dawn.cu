// dawn.cu — C ABI (include/dawn.h) over the sm_100a weighted-DAWN kernels.
//
// Memory model: the graph and each solver's workspace are allocated once
// (from the device memory pool, outside any solve); a solve performs no allocation.  Device
// layout per graph (32-bit indices when m < 2^32):
//   row_ptr : EI[n+1]
//   edges   : uint2 {col, weight bits}[m]        (4-byte value types: 8 B/edge, one LDG.64)
//             uint32 col[m] + uint64 w[m]         (8-byte value types: 12 B/edge)
// Per solver: dist keys K[n], write stamps u32[n], two frontier queues
// {node u32, off EI, base EI, key K}[n], a tile->row map u32[m/TILE+2], and
// the DevState block.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <charconv>
#include <type_traits>
#include <climits>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/dawn.h"
#include "dawn_batch.cuh"
#include "dawn_csr.cuh"
#include "dawn_fw.cuh"
#include "dawn_nearfar.cuh"
#include "dawn_small.cuh"

using namespace dawn;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      return fail(e_ == cudaErrorMemoryAllocation ? DAWN_ENOMEM : DAWN_ECUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                     \
    }                                                                                     \
  } while (0)

#define TRY(expr)              \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != DAWN_OK) return rc_; \
  } while (0)

// ---------------------------------------------------------------------------
// memory: device buffers come from the device's stream-ordered pool with an
// unbounded release threshold, so creating and destroying graphs / solvers of
// the same sizes (a plugin handle per call, the e2e bench step) reuses memory
// instead of paying cudaMalloc + cudaFree (~16 ms for a config-2 solver).
// Frees follow a device synchronisation, as cudaFree's implicit one did.
// Small pinned host blocks (state read-back) are cached the same way.
// ---------------------------------------------------------------------------
static std::mutex g_mem_mu;
static bool g_pool_ready[128];

static cudaError_t dmalloc_raw(void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(g_mem_mu);
    if (dev >= 0 && dev < 128 && !g_pool_ready[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      g_pool_ready[dev] = true;
    }
  }
  e = cudaMallocAsync(p, bytes, 0);
  if (e != cudaSuccess) {
    *p = nullptr;
    return e;
  }
  return cudaStreamSynchronize(0);  // usable from any stream from here on
}
template <class T>
static cudaError_t dmalloc(T** p, size_t bytes) {
  return dmalloc_raw(reinterpret_cast<void**>(p), bytes);
}
static void dfree(void* p) {
  if (p) cudaFreeAsync(p, 0);
}

static std::vector<std::pair<size_t, void*>> g_host_free;  // cached pinned blocks (size, ptr)
template <class T>
static cudaError_t hmalloc(T** p, size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_mem_mu);
    for (size_t i = 0; i < g_host_free.size(); ++i) {
      if (g_host_free[i].first == bytes) {
        *p = reinterpret_cast<T*>(g_host_free[i].second);
        g_host_free.erase(g_host_free.begin() + (long)i);
        return cudaSuccess;
      }
    }
  }
  void* q = nullptr;
  cudaError_t e = cudaMallocHost(&q, bytes + 16);  // + 16: the block remembers its size
  if (e != cudaSuccess) return e;
  *reinterpret_cast<size_t*>(q) = bytes;
  *p = reinterpret_cast<T*>(reinterpret_cast<char*>(q) + 16);
  return cudaSuccess;
}
static void hfree(void* p) {
  if (!p) return;
  char* q = reinterpret_cast<char*>(p) - 16;
  std::lock_guard<std::mutex> lk(g_mem_mu);
  if (g_host_free.size() < 64) g_host_free.emplace_back(*reinterpret_cast<size_t*>(q), p);
  else cudaFreeHost(q);
}

// ---------------------------------------------------------------------------
// objects
// ---------------------------------------------------------------------------
struct dawn_graph_s {
  int device = 0;
  int64_t n = 0, m = 0;
  int vtype = DAWN_F64;
  bool wide = false;      // 64-bit edge indices
  bool has_negative = false;
  void* row_ptr = nullptr;
  uint2* e2 = nullptr;
  uint32_t* ecol = nullptr;
  unsigned long long* ew = nullptr;
  int64_t bytes = 0;
};

struct dawn_solver_s {
  dawn_graph_t g = nullptr;
  unsigned flags = 0;
  void* dist = nullptr;
  uint32_t* stamp = nullptr;
  uint32_t* bmap = nullptr;      // bitmap frontier (low-degree graphs)
  uint8_t* wstate = nullptr;
  unsigned long long* pred = nullptr;
  uint32_t* jmp0 = nullptr;
  uint32_t* jmp1 = nullptr;
  uint32_t* qnode[2] = {nullptr, nullptr};
  void* qoff[2] = {nullptr, nullptr};
  void* qbase[2] = {nullptr, nullptr};
  void* qkey[2] = {nullptr, nullptr};
  uint32_t* tile_row = nullptr;
  unsigned long long* wl_ring = nullptr;  // worklist tail (graphs without negative weights)
  uint64_t wl_cap = 0;
  int wl_grid = 1;
  double worklist_edges = 1 << 20;        // tunable: async rounds relaxing < this many edges end the solve barrier-free (0 = off)
  DevState* st = nullptr;
  DevState* st_host = nullptr;  // pinned
  double* dbuf = nullptr;
  int64_t* pbuf = nullptr;
  unsigned long long* prof = nullptr;  // per-round timeline (DAWN_F_PROFILE)
  unsigned long long* cta_prof = nullptr;  // debug per-CTA phase ends (DAWN_F_PROFILE, 256 rounds)
  unsigned prof_cap = 0;
  int grid = 1;       // co-resident CTAs of the plain persistent kernel
  int grid_pred = 1;  // ... of the predecessor-tracking instance
  size_t smem = 0;
  double dense_edges_per_node = 0.5;  // tunable: dense frontier build after rounds relaxing >= this * n edges
  uint32_t* phist = nullptr;          // priority window histograms [2][PW_BINS]
  double pw_frac = 0.2;               // tunable "priority_frac": heavy async rounds relax the lowest this share
                                      // of the frontier's edges by row value (0 = off)
  double pw_edges_per_edge = 0.4;     // tunable "priority_edges_per_edge": ... rounds relaxing >= this * m edges
  double pw_seed_edges = 4096;        // tunable "priority_seed_edges": a source row this long windows round 2 too
  int wide_pref = -1;                 // tunable "wide_tiles": -1 auto, 0 narrow, 1 wide X-phase tiles
  bool wide = false;
  int fb_pref = -1;                   // tunable "bitmap_frontier": -1 auto, 0 off, 1 on
  bool fb = false;
  int nf_pref = -1;                   // tunable "nearfar": -1 auto (low-degree graphs), 0 off, 1 on
  bool nf = false;                    // async solves without negative weights run dawn_nearfar
  double nf_delta = 0;                // tunable "nearfar_delta": bucket width in weight units (0 = auto)
  double nf_delta_mean = 8;           // tunable "nearfar_delta_mean": auto width = this * mean edge weight
  double mean_w = -1;                 // mean edge weight (computed on first near-far solve)
  double nf_cap = 64;                 // tunable "nearfar_batches": continuation batches per warp per round
  int nf_grid = 1;
  int small_pref = -1;                // tunable "small_graph": -1 auto, 0 off, 1 on (when it fits)
  bool small = false;                 // unbounded solves without negative weights run dawn_small (one CTA)
  int small_cl = 0;                   // its cluster size (CTAs)
  int small_cl_max = SM_MAXCL;        // tunable "small_cluster": largest cluster to try (power of two)
  size_t small_smem = 0;
  bool init_pending = false;          // begin deferred to the small kernel (see Impl::begin)
  bool spec = true;                   // tunable "speculate_negcheck": negative-weight solves try the plain kernel first
  double batch_min_sources = 4;       // tunable: dawn_mssp batches when k >= this
  double batch_sparse_util = 4;       // tunable: batched rounds averaging < this active sources per edge go lane-sparse
  int ebits = 32;
  int logn = 0;
  // batched multi-source workspace (allocated on first use, kept)
  bool batch_ready = false;
  bool last_batch = false;       // the last solve on this solver was a batch (round profile source)
  void* bd = nullptr;            // K[n][32]
  uint32_t* bmask[4] = {nullptr, nullptr, nullptr, nullptr};  // nmask, w1, w2, smask
  uint32_t* bqnode[2] = {nullptr, nullptr};  // row lists 0 (whole line) and 1 (lane by lane)
  uint32_t* bqmask[2] = {nullptr, nullptr};
  void* bqoff[2] = {nullptr, nullptr};
  void* bqbase[2] = {nullptr, nullptr};
  void* bqkey = nullptr;         // K[n][32]
  uint32_t* btile[2] = {nullptr, nullptr};
  BState* bst = nullptr;
  BState* bst_host = nullptr;    // pinned, one per batch in flight
  int64_t bst_host_cap = 0;
  void* bout = nullptr;          // double[32][n] staging for host outputs
  int bgrid = 1;
  size_t bsmem = 0;
  // current solve
  int64_t source = -1;
  int algo = 0;
  unsigned run_flags = 0;
  bool active = false;
};

static int bitlen(uint64_t x) {
  int b = 0;
  while (x) { ++b; x >>= 1; }
  return b;
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// page-locked host memory the device can read in place (UVA): the upload
// kernels stream it over PCIe without a staging copy
static bool is_pinned_host_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
}

// ---------------------------------------------------------------------------
// graph upload / conversion kernels
// ---------------------------------------------------------------------------
enum : unsigned { ERR_COL = 1u, ERR_NONINT = 2u, ERR_RANGE = 4u, NEG = 8u, ERR_ROWPTR = 16u };

template <class V>
__global__ void k_convert_edges(const int64_t* __restrict__ col, const double* __restrict__ val,
                                int64_t m, int64_t n, uint2* __restrict__ e2,
                                uint32_t* __restrict__ ecol, unsigned long long* __restrict__ ew,
                                unsigned* flags) {
  unsigned f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = col[i];
    if (c < 0 || c >= n) f |= ERR_COL;
    const double w = val[i];
    if (w < 0) f |= NEG;
    if constexpr (sizeof(V) == 4) {
      uint32_t wb;
      if constexpr (std::is_same<V, int32_t>::value) {
        if (w != rint(w)) f |= ERR_NONINT;
        if (!(fabs(w) <= 2147483647.0)) f |= ERR_RANGE;
        wb = (uint32_t)(int32_t)w;
      } else {
        float x = (float)w;
        if (isinf(x)) f |= ERR_RANGE;
        wb = __float_as_uint(x);
      }
      e2[i] = make_uint2((uint32_t)c, wb);
    } else {
      unsigned long long wb;
      if constexpr (std::is_same<V, int64_t>::value) {
        if (w != rint(w)) f |= ERR_NONINT;
        if (!(fabs(w) < 9223372036854775807.0)) f |= ERR_RANGE;
        wb = (unsigned long long)(long long)w;
      } else {
        wb = (unsigned long long)__double_as_longlong(w);
      }
      ecol[i] = (uint32_t)c;
      ew[i] = wb;
    }
  }
  if (f) atomicOr(flags, f);
}

template <class EI>
__global__ void k_convert_rowptr(const int64_t* __restrict__ rp, int64_t n, int64_t m,
                                 EI* __restrict__ out, unsigned* flags) {
  unsigned f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = rp[i];
    if (i == 0 && a != 0) f |= ERR_ROWPTR;
    if (i == n && a != m) f |= ERR_ROWPTR;
    if (i < n && rp[i + 1] < a) f |= ERR_ROWPTR;
    out[i] = (EI)a;
  }
  if (f) atomicOr(flags, f);
}

static int value_size(int vtype) { return (vtype == DAWN_I32 || vtype == DAWN_F32) ? 4 : 8; }

extern "C" int dawn_abi_version(void) { return DAWN_ABI_VERSION; }
extern "C" const char* dawn_last_error(void) { return g_last_error.c_str(); }

extern "C" int dawn_device_count(int* count_out) {
  if (!count_out) return fail(DAWN_EINVAL, "count_out is NULL");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count_out = 0;
    return fail(DAWN_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count_out = c;
  return DAWN_OK;
}

extern "C" int dawn_choose_vtype(int64_t n, int64_t m, const double* val, int precision,
                                 int* vtype_out) {
  if (!vtype_out || n < 0 || m < 0 || (m > 0 && !val)) return fail(DAWN_EINVAL, "bad arguments");
  if (precision == DAWN_PREC_FP32) { *vtype_out = DAWN_F32; return DAWN_OK; }
  if (precision == DAWN_PREC_FP64) { *vtype_out = DAWN_F64; return DAWN_OK; }
  if (precision != DAWN_PREC_AUTO) return fail(DAWN_EINVAL, "unknown precision %d", precision);
  bool integral = true;
  double maxabs = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    const double w = val[i];
    if (!isfinite(w)) return fail(DAWN_EINVAL, "weights must be finite");
    if (integral && w != floor(w)) integral = false;
    maxabs = std::max(maxabs, fabs(w));
  }
  if (!integral) { *vtype_out = DAWN_F64; return DAWN_OK; }
  // |dist| after r rounds is at most r*max|w| with r <= n; one more edge for the candidate.
  const double bound = ((double)n + 1.0) * maxabs;
  if (bound < 2147483647.0) *vtype_out = DAWN_I32;
  else if (bound < 9007199254740992.0) *vtype_out = DAWN_I64;  // 2^53: reference fp64 sums exact
  else *vtype_out = DAWN_F64;
  return DAWN_OK;
}

template <class V>
static int convert_graph(dawn_graph_t g, const int64_t* d_rp, const int64_t* d_col,
                         const double* d_val, unsigned* d_flags) {
  const int64_t n = g->n, m = g->m;
  const int blocks = 148 * 8;
  if (g->wide) {
    k_convert_rowptr<unsigned long long><<<blocks, 256>>>(d_rp, n, m, (unsigned long long*)g->row_ptr, d_flags);
  } else {
    k_convert_rowptr<uint32_t><<<blocks, 256>>>(d_rp, n, m, (uint32_t*)g->row_ptr, d_flags);
  }
  CK(cudaGetLastError());
  if (m > 0) {
    k_convert_edges<V><<<blocks, 256>>>(d_col, d_val, m, n, g->e2, g->ecol, g->ew, d_flags);
    CK(cudaGetLastError());
  }
  return DAWN_OK;
}

// Host-resident inputs of real size: the edge arrays cross PCIe by DMA in
// chunks into two device staging slots while the previous chunk converts on a
// second stream (copy engine and SMs overlap; zero-copy reads of pinned memory
// reached ~51 GB/s against ~55 GB/s for the DMA).
template <class V>
static int convert_graph_staged(dawn_graph_t g, const int64_t* h_rp, const int64_t* h_col, const double* h_val,
                                unsigned* d_flags) {
  const int64_t n = g->n, m = g->m;
  constexpr int64_t CHE = 1ll << 22;  // edges per chunk (64 MB of col + val)
  const int blocks = 148 * 8;
  char* stage = nullptr;
  const size_t slot = 16 * (size_t)std::min<int64_t>(CHE, m);
  CK(dmalloc(&stage, 8 * (size_t)(n + 1) + 2 * slot));
  cudaStream_t cs = nullptr, ks = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
  auto finish = [&](int rc) {
    if (ks) cudaStreamSynchronize(ks);
    if (cs) cudaStreamSynchronize(cs);
    for (int i = 0; i < 2; ++i) {
      if (copied[i]) cudaEventDestroy(copied[i]);
      if (used[i]) cudaEventDestroy(used[i]);
    }
    if (cs) cudaStreamDestroy(cs);
    if (ks) cudaStreamDestroy(ks);
    dfree(stage);
    return rc;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking)) != cudaSuccess)
    return finish(fail(DAWN_ECUDA, "streams: %s", cudaGetErrorString(e)));
  for (int i = 0; i < 2; ++i)
    if ((e = cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&used[i], cudaEventDisableTiming)) != cudaSuccess)
      return finish(fail(DAWN_ECUDA, "events: %s", cudaGetErrorString(e)));
  // the flags were cleared on the legacy stream, which these non-blocking streams do not follow
  if ((e = cudaStreamSynchronize(0)) != cudaSuccess)
    return finish(fail(DAWN_ECUDA, "graph upload: %s", cudaGetErrorString(e)));
  // row pointers first (the monotonicity check reads the whole array)
  int64_t* s_rp = (int64_t*)stage;
  if ((e = cudaMemcpyAsync(s_rp, h_rp, 8 * (size_t)(n + 1), cudaMemcpyHostToDevice, ks)) != cudaSuccess)
    return finish(fail(DAWN_ECUDA, "graph upload: %s", cudaGetErrorString(e)));
  if (g->wide)
    k_convert_rowptr<unsigned long long><<<blocks, 256, 0, ks>>>(s_rp, n, m, (unsigned long long*)g->row_ptr, d_flags);
  else
    k_convert_rowptr<uint32_t><<<blocks, 256, 0, ks>>>(s_rp, n, m, (uint32_t*)g->row_ptr, d_flags);
  char* slots = stage + 8 * (size_t)(n + 1);
  for (int64_t off = 0, c = 0; off < m; off += CHE, ++c) {
    const int64_t len = std::min<int64_t>(CHE, m - off);
    const int b = (int)(c & 1);
    int64_t* s_col = (int64_t*)(slots + b * slot);
    double* s_val = (double*)(s_col + std::min<int64_t>(CHE, m));
    if (c >= 2 && (e = cudaStreamWaitEvent(cs, used[b], 0)) != cudaSuccess)
      return finish(fail(DAWN_ECUDA, "graph upload: %s", cudaGetErrorString(e)));
    if ((e = cudaMemcpyAsync(s_col, h_col + off, 8 * (size_t)len, cudaMemcpyHostToDevice, cs)) != cudaSuccess ||
        (e = cudaMemcpyAsync(s_val, h_val + off, 8 * (size_t)len, cudaMemcpyHostToDevice, cs)) != cudaSuccess ||
        (e = cudaEventRecord(copied[b], cs)) != cudaSuccess || (e = cudaStreamWaitEvent(ks, copied[b], 0)) != cudaSuccess)
      return finish(fail(DAWN_ECUDA, "graph upload: %s", cudaGetErrorString(e)));
    k_convert_edges<V><<<blocks, 256, 0, ks>>>(s_col, s_val, len, n, g->e2 ? g->e2 + off : nullptr,
                                               g->ecol ? g->ecol + off : nullptr, g->ew ? g->ew + off : nullptr,
                                               d_flags);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaEventRecord(used[b], ks)) != cudaSuccess)
      return finish(fail(DAWN_ECUDA, "graph convert: %s", cudaGetErrorString(e)));
  }
  return finish(DAWN_OK);
}

static void graph_free(dawn_graph_t g) {
  if (!g) return;
  cudaSetDevice(g->device);
  cudaDeviceSynchronize();
  dfree(g->row_ptr);
  dfree(g->e2);
  dfree(g->ecol);
  dfree(g->ew);
  delete g;
}

extern "C" int dawn_graph_create(int device, int64_t n, int64_t m, const int64_t* row_ptr,
                                 const int64_t* col, const double* val, int vtype,
                                 int src_is_device, dawn_graph_t* out) {
  if (!out) return fail(DAWN_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || m < 0 || !row_ptr || (m > 0 && (!col || !val)))
    return fail(DAWN_EINVAL, "bad graph arguments (n=%lld, m=%lld)", (long long)n, (long long)m);
  if (vtype < DAWN_I32 || vtype > DAWN_F64) return fail(DAWN_EINVAL, "unknown vtype %d", vtype);
  if ((uint64_t)n >= 0xFFFFFFFEull || n >= (1ll << 31))
    return fail(DAWN_EUNSUPPORTED, "n=%lld exceeds the 2^31 node limit", (long long)n);
  const int cbits = bitlen((uint64_t)n);
  if (bitlen((uint64_t)m) >= 64 - cbits)
    return fail(DAWN_EUNSUPPORTED, "m=%lld too large for the packed frontier reservation", (long long)m);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(DAWN_EINVAL, "device %d out of range (%d devices)", device, ndev);
  CK(cudaSetDevice(device));

  dawn_graph_s* g = new dawn_graph_s();
  g->device = device;
  g->n = n;
  g->m = m;
  g->vtype = vtype;
  g->wide = (uint64_t)m > 0xFFFFFFFFull - 4ull * TILE;
  const size_t eis = g->wide ? 8 : 4;
  auto cleanup = [&](int rc) { graph_free(g); return rc; };
  cudaError_t e;
  if ((e = dmalloc(&g->row_ptr, eis * (size_t)(n + 1))) != cudaSuccess)
    return cleanup(fail(DAWN_ENOMEM, "row_ptr alloc: %s", cudaGetErrorString(e)));
  g->bytes += eis * (n + 1);
  const size_t mm = (size_t)std::max<int64_t>(m, 1);
  if (value_size(vtype) == 4) {
    if ((e = dmalloc(&g->e2, 8 * mm)) != cudaSuccess)
      return cleanup(fail(DAWN_ENOMEM, "edge alloc: %s", cudaGetErrorString(e)));
    g->bytes += 8 * mm;
  } else {
    if ((e = dmalloc(&g->ecol, 4 * mm)) != cudaSuccess ||
        (e = dmalloc(&g->ew, 8 * mm)) != cudaSuccess)
      return cleanup(fail(DAWN_ENOMEM, "edge alloc: %s", cudaGetErrorString(e)));
    g->bytes += 12 * mm;
  }

  // stage the reference-layout arrays on the device if they live on the host
  const int64_t* d_rp = row_ptr;
  const int64_t* d_col = col;
  const double* d_val = val;
  void* tmp = nullptr;
  unsigned* d_flags = nullptr;
  const bool pinned = !src_is_device && is_pinned_host_ptr(row_ptr) && (m == 0 || (is_pinned_host_ptr(col) &&
                                                                                   is_pinned_host_ptr(val)));
  const bool staged = !src_is_device && m >= (1ll << 22);  // large host graphs: chunked DMA + convert
  if (staged) {
    // converted below by convert_graph_staged
  } else if (pinned) {
    cudaPointerAttributes a;
    cudaPointerGetAttributes(&a, row_ptr);
    d_rp = (const int64_t*)a.devicePointer;
    if (m) {
      cudaPointerGetAttributes(&a, col);
      d_col = (const int64_t*)a.devicePointer;
      cudaPointerGetAttributes(&a, val);
      d_val = (const double*)a.devicePointer;
    }
  } else if (!src_is_device) {
    const size_t bytes = 8 * (size_t)(n + 1) + 16 * (size_t)m;
    if ((e = dmalloc(&tmp, bytes)) != cudaSuccess)
      return cleanup(fail(DAWN_ENOMEM, "staging alloc: %s", cudaGetErrorString(e)));
    char* p = (char*)tmp;
    int64_t* s_rp = (int64_t*)p;
    int64_t* s_col = (int64_t*)(p + 8 * (n + 1));
    double* s_val = (double*)(p + 8 * (n + 1) + 8 * m);
    e = cudaMemcpy(s_rp, row_ptr, 8 * (size_t)(n + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && m) e = cudaMemcpy(s_col, col, 8 * (size_t)m, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && m) e = cudaMemcpy(s_val, val, 8 * (size_t)m, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      dfree(tmp);
      return cleanup(fail(DAWN_ECUDA, "graph upload: %s", cudaGetErrorString(e)));
    }
    d_rp = s_rp;
    d_col = s_col;
    d_val = s_val;
  }
  if ((e = dmalloc(&d_flags, sizeof(unsigned))) != cudaSuccess ||
      (e = cudaMemset(d_flags, 0, sizeof(unsigned))) != cudaSuccess) {
    dfree(tmp);
    return cleanup(fail(DAWN_ECUDA, "flags: %s", cudaGetErrorString(e)));
  }
  int rc = DAWN_OK;
  if (staged) {
    switch (vtype) {
      case DAWN_I32: rc = convert_graph_staged<int32_t>(g, row_ptr, col, val, d_flags); break;
      case DAWN_I64: rc = convert_graph_staged<int64_t>(g, row_ptr, col, val, d_flags); break;
      case DAWN_F32: rc = convert_graph_staged<float>(g, row_ptr, col, val, d_flags); break;
      default: rc = convert_graph_staged<double>(g, row_ptr, col, val, d_flags); break;
    }
  } else {
    switch (vtype) {
      case DAWN_I32: rc = convert_graph<int32_t>(g, d_rp, d_col, d_val, d_flags); break;
      case DAWN_I64: rc = convert_graph<int64_t>(g, d_rp, d_col, d_val, d_flags); break;
      case DAWN_F32: rc = convert_graph<float>(g, d_rp, d_col, d_val, d_flags); break;
      default: rc = convert_graph<double>(g, d_rp, d_col, d_val, d_flags); break;
    }
  }
  unsigned hflags = 0;
  if (rc == DAWN_OK) {
    e = cudaMemcpy(&hflags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(DAWN_ECUDA, "graph convert: %s", cudaGetErrorString(e));
  }
  dfree(tmp);
  dfree(d_flags);
  if (rc != DAWN_OK) return cleanup(rc);
  if (hflags & ERR_ROWPTR) return cleanup(fail(DAWN_EINVAL, "row_ptr must start at 0, end at m and be monotone"));
  if (hflags & ERR_COL) return cleanup(fail(DAWN_EINVAL, "column index out of range"));
  if (hflags & ERR_NONINT) return cleanup(fail(DAWN_EINVAL, "non-integral weight for an integer value type"));
  if (hflags & ERR_RANGE) return cleanup(fail(DAWN_EINVAL, "weight out of range for the value type"));
  g->has_negative = (hflags & NEG) != 0;
  *out = g;
  return DAWN_OK;
}

extern "C" int dawn_graph_destroy(dawn_graph_t g) {
  graph_free(g);
  return DAWN_OK;
}

extern "C" int dawn_graph_info(dawn_graph_t g, int64_t* n, int64_t* m, int* vtype,
                               int64_t* device_bytes) {
  if (!g) return fail(DAWN_EINVAL, "graph is NULL");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (vtype) *vtype = g->vtype;
  if (device_bytes) *device_bytes = g->bytes;
  return DAWN_OK;
}

// ---------------------------------------------------------------------------
// solver
// ---------------------------------------------------------------------------
template <class V, class EI>
struct Impl {
  using K = typename Val<V>::K;

  static KParams<V, EI> params(dawn_solver_t s, unsigned max_rounds) {
    dawn_graph_t g = s->g;
    KParams<V, EI> P;
    P.n = (uint32_t)g->n;
    P.src = (uint32_t)s->source;
    P.row_ptr = (const EI*)g->row_ptr;
    P.e2 = g->e2;
    P.ecol = g->ecol;
    P.ew = g->ew;
    P.dist = (K*)s->dist;
    P.stamp = s->stamp;
    P.bmap = s->bmap;
    P.wstate = s->wstate;
    P.pred = s->pred;
    P.jmp0 = s->jmp0;
    P.jmp1 = s->jmp1;
    for (int i = 0; i < 2; ++i) {
      P.qnode[i] = s->qnode[i];
      P.qoff[i] = (EI*)s->qoff[i];
      P.qbase[i] = (EI*)s->qbase[i];
      P.qkey[i] = (K*)s->qkey[i];
    }
    P.tile_row = s->tile_row;
    P.st = s->st;
    P.algo = s->algo;
    const bool neg = (s->run_flags & DAWN_F_NEGCHECK) && g->has_negative &&
                     (g->vtype == DAWN_I32 || g->vtype == DAWN_I64) && s->pred != nullptr;
    P.pred_on = ((s->run_flags & DAWN_F_PRED) || neg) ? 1 : 0;
    P.negcheck_period = neg ? 16 : 0;
    P.logn = s->logn;
    P.ebits = s->ebits;
    P.max_rounds = max_rounds;
    P.dense_edges = (unsigned long long)std::max(1.0, s->dense_edges_per_node * (double)g->n);
    P.prof = s->prof;
    P.prof_cap = s->prof_cap;
    P.cta_prof = s->cta_prof;
    P.live = (s->run_flags & DAWN_F_ASYNC) && !P.pred_on ? 1 : 0;
    P.wl_ring = s->worklist_edges > 0 ? s->wl_ring : nullptr;
    P.wl_mask = s->wl_cap ? s->wl_cap - 1 : 0;
    P.wl_edges = (unsigned long long)s->worklist_edges;
    P.nf_delta = s->nf_delta > 0 ? s->nf_delta : s->nf_delta_mean * std::max(s->mean_w, 0.0);
    if (!(P.nf_delta > 0)) P.nf_delta = std::is_floating_point<V>::value ? 1e-3 : 1.0;
    P.nf_cap = (uint32_t)std::min(s->nf_cap, 4.0e9);
    P.skip_if_done = 0;
    P.phist = s->phist;
    P.pw_frac = (float)s->pw_frac;
    P.pw_edges = std::max(P.dense_edges, (unsigned long long)std::max(1.0, s->pw_edges_per_edge * (double)g->m));
    P.pw_seed_edges = (unsigned long long)std::min(std::max(1.0, s->pw_seed_edges), 1.8e19);
    P.pw = (P.live && P.algo == 0 && !g->has_negative && sizeof(K) == 4 && !P.pred_on && !s->fb &&
            max_rounds == 0xFFFFFFFFu && s->phist != nullptr && s->pw_frac > 0.0 && s->pw_frac < 1.0) ? 1 : 0;
    return P;
  }

  // tile width of the X phase: wide (XI_WIDE edges per lane) for 4-byte values
  // on graphs with heavy rounds, narrow (8) otherwise
  static constexpr int XW = sizeof(K) == 4 ? XI_WIDE : XI_NARROW;
  template <int XI>
  static void* kernel(bool pred, bool raw) {
    if (pred) return raw ? (void*)dawn_persistent<V, EI, true, true, XI> : (void*)dawn_persistent<V, EI, true, false, XI>;
    return raw ? (void*)dawn_persistent<V, EI, false, true, XI> : (void*)dawn_persistent<V, EI, false, false, XI>;
  }
  static void* kernel_for(dawn_solver_t s, bool pred) {
    const bool raw = !s->g->has_negative;
    if (!pred && s->fb)  // bitmap-frontier variant (narrow tiles, no predecessor pass)
      return raw ? (void*)dawn_persistent<V, EI, false, true, XI_NARROW, true>
                 : (void*)dawn_persistent<V, EI, false, false, XI_NARROW, true>;
    return s->wide ? kernel<XW>(pred, raw) : kernel<XI_NARROW>(pred, raw);
  }

  // mean edge weight (the near-far bucket width is a multiple of it); once per solver
  static int mean_weight(dawn_solver_t s, cudaStream_t stream) {
    const int64_t m = s->g->m;
    double* d = nullptr;
    CK(dmalloc(&d, sizeof(double)));
    CK(cudaMemsetAsync(d, 0, sizeof(double), stream));
    if (m > 0) {
      const int blocks = (int)std::min<int64_t>(148 * 4, (m + 255) / 256);
      dawn_weight_sum<V><<<blocks, 256, 0, stream>>>(s->g->e2, s->g->ew, (uint64_t)m, d);
      CK(cudaGetLastError());
    }
    double h = 0;
    CK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    dfree(d);
    s->mean_w = m > 0 ? h / (double)m : 0.0;
    return DAWN_OK;
  }

  static int setup(dawn_solver_t s) {
    const int64_t n = s->g->n, m = s->g->m;
    if (s->wide_pref < 0) s->wide = XW != XI_NARROW && m >= (1ll << 25) && m >= 8 * n;
    else s->wide = XW != XI_NARROW && s->wide_pref > 0;
    // low-degree graphs (average out-degree < 8, e.g. grids / road networks):
    // light rounds keep a bitmap frontier instead of enqueueing every write
    if (s->fb_pref < 0) s->fb = !s->wide && m < 8 * n && n >= 4096;
    else s->fb = !s->wide && s->fb_pref > 0;
    const size_t sm = s->wide ? sizeof(Smem<V, EI, XW>) : sizeof(Smem<V, EI, XI_NARROW>);
    const void* k0 = kernel_for(s, false);
    const void* k1 = kernel_for(s, true);
    if (s->fb) {  // the predecessor-tracking instance stays on the queue frontier
      const bool raw = !s->g->has_negative;
      const void* kq = s->wide ? kernel<XW>(false, raw) : kernel<XI_NARROW>(false, raw);
      CK(cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    CK(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    // Keep the shared-memory carveout to what DAWN_MIN_BLOCKS resident CTAs
    // need: the rest of the unified 228 KB stays L1, which serves the skewed
    // dist[] gathers (an L2-only gather caps the relax at ~140 G edges/s).
    {
      const double need_kb = DAWN_MIN_BLOCKS * ((double)sm / 1024.0 + 1.0);
      const int pct = std::min(100, (int)std::ceil(100.0 * need_kb / 228.0));
      CK(cudaFuncSetAttribute(k0, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
      CK(cudaFuncSetAttribute(k1, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    }
    int bps0 = 0, bps1 = 0, nsm = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps0, k0, NT, sm));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps1, k1, NT, sm));
    if (bps0 < 1 || bps1 < 1) return fail(DAWN_ECUDA, "persistent kernel cannot be resident (smem %zu)", sm);
    const int64_t work = std::max<int64_t>((n + TILE - 1) / TILE, (m + TILE - 1) / TILE);
    s->grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)bps0 * nsm, work));
    s->grid_pred = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)bps1 * nsm, work));
    s->smem = sm;
    int bpw = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpw, dawn_worklist<V, EI>, NT, 0));
    s->wl_grid = std::max(1, bpw) * nsm;
    // small graphs: one thread-block cluster with the solve state in distributed
    // shared memory (no negative weights)
    s->small = false;
    if (!s->g->has_negative && s->small_pref != 0 && n >= 2 && m < (1ll << 31)) {
      int optin = 0;
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      const int dyn_max = optin - 4096;  // static shared memory of the kernel stays below 4 KB
      for (auto fn : {(const void*)dawn_small<V, EI, false>, (const void*)dawn_small<V, EI, true>}) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      }
      s->small_cl = 0;
      for (int cl = s->small_cl_max; cl >= 1 && !s->small_cl; cl >>= 1) {
        const size_t need = small_smem_bytes<V, EI>((uint32_t)n, (uint32_t)cl);
        if (need > (size_t)dyn_max) break;  // a smaller cluster needs even more per CTA
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(SM_NT);
        cfg.dynamicSmemBytes = need;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, (const void*)dawn_small<V, EI, false>, &cfg) == cudaSuccess && nc > 0) {
          s->small_cl = cl;
          s->small_smem = need;
        }
        cudaGetLastError();
      }
      // auto: graphs whose rounds are latency-bound on the grid (config 1: 16 K nodes)
      s->small = s->small_cl > 0 && (s->small_pref > 0 || (n <= (1 << 16) && m <= (1ll << 18)));
    }
    // near-far schedule (async, no negative weights): on by default where the bitmap frontier is
    s->nf = s->nf_pref < 0 ? s->fb : s->nf_pref > 0;
    int bpn = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpn, dawn_nearfar<V, EI>, NT, 0));
    if (bpn < 1) return fail(DAWN_ECUDA, "near-far kernel cannot be resident");
    const int64_t chunks = ((n + 31) / 32 + 127) / 128;  // 128-word sweep chunks, one per warp
    s->nf_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::min(bpn, DAWN_MIN_BLOCKS) * nsm,
                                                            (chunks + WPB - 1) / WPB));
    return DAWN_OK;
  }

  // the small-graph cluster kernel initialises its own state: its solves skip
  // the begin kernel unless something else (stepping, a state read) runs first
  static int begin(dawn_solver_t s, cudaStream_t stream) {
    s->init_pending = false;
    if (s->small && !(s->run_flags & DAWN_F_PRED) && !s->g->has_negative && !s->prof &&
        !nearfar_eligible(s, 0xFFFFFFFFu)) {
      s->init_pending = true;
      return DAWN_OK;
    }
    return init_solve(s, stream);
  }

  static int init_solve(dawn_solver_t s, cudaStream_t stream) {
    s->init_pending = false;
    const int64_t n = s->g->n;
    if (s->prof) CK(cudaMemsetAsync(s->prof, 0, 32 * (size_t)s->prof_cap, stream));
    if (s->pred) CK(cudaMemsetAsync(s->pred, 0, sizeof(unsigned long long) * n, stream));
    KParams<V, EI> P = params(s, 0);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + 255) / 256));
    if (s->g->has_negative) dawn_begin_solve<V, EI, false><<<blocks, 256, 0, stream>>>(P);
    else dawn_begin_solve<V, EI, true><<<blocks, 256, 0, stream>>>(P);
    CK(cudaGetLastError());
    return DAWN_OK;
  }

  static bool nearfar_eligible(dawn_solver_t s, unsigned max_rounds) {
    return s->nf && (s->run_flags & DAWN_F_ASYNC) && !(s->run_flags & DAWN_F_PRED) && s->algo == DAWN_GOVM &&
           max_rounds == 0xFFFFFFFFu && !s->g->has_negative;
  }

  static int run(dawn_solver_t s, unsigned max_rounds, cudaStream_t stream) {
    // async on low-degree graphs: the near-far schedule (far less work than any round schedule)
    const bool nf = nearfar_eligible(s, max_rounds);
    if (s->small && !nf && max_rounds == 0xFFFFFFFFu && !(s->run_flags & DAWN_F_PRED) &&
        !s->g->has_negative) {
      s->init_pending = false;
      KParams<V, EI> P = params(s, max_rounds);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(s->small_cl);
      cfg.blockDim = dim3(SM_NT);
      cfg.dynamicSmemBytes = s->small_smem;
      cfg.stream = stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = s->small_cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (s->run_flags & DAWN_F_ASYNC) CK(cudaLaunchKernelEx(&cfg, dawn_small<V, EI, true>, P));
      else CK(cudaLaunchKernelEx(&cfg, dawn_small<V, EI, false>, P));
      return DAWN_OK;
    }
    if (s->init_pending) TRY(init_solve(s, stream));
    // Integer graphs with negative weights run the predecessor-tracking kernel
    // (a second relax pass per round) only for the cycle check every
    // negcheck_period rounds.  Speculate first: the plain kernel runs the same
    // rounds up to the first check; a solve that converges by then (no
    // negative cycle: the common case, config 5a) is finished and the two
    // launches behind it return at once; otherwise the state is reset on the
    // device and the tracking kernel solves from scratch.  No host sync.
    {
      KParams<V, EI> P = params(s, max_rounds);
      if (P.negcheck_period > 0 && !(s->run_flags & DAWN_F_PRED) && max_rounds == 0xFFFFFFFFu && s->spec) {
        KParams<V, EI> Q = P;
        Q.pred_on = 0;
        Q.negcheck_period = 0;
        Q.live = 0;
        Q.wl_ring = nullptr;
        Q.max_rounds = (unsigned)P.negcheck_period;
        void* qa[] = {&Q};
        CK(cudaLaunchCooperativeKernel(kernel_for(s, false), dim3(s->grid), dim3(NT), qa, s->smem, stream));
        KParams<V, EI> B = P;
        B.skip_if_done = 1;
        const int64_t n = s->g->n;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + 255) / 256));
        dawn_begin_solve<V, EI, false><<<blocks, 256, 0, stream>>>(B);  // negative weights: sign-flip keys
        CK(cudaGetLastError());
        P.skip_if_done = 1;
        void* pa[] = {&P};
        CK(cudaLaunchCooperativeKernel(kernel_for(s, true), dim3(s->grid_pred), dim3(NT), pa, s->smem, stream));
        return DAWN_OK;
      }
    }
    if (nearfar_eligible(s, max_rounds)) {
      if (s->mean_w < 0) TRY(mean_weight(s, stream));
      KParams<V, EI> P = params(s, max_rounds);
      void* args[] = {&P};
      CK(cudaLaunchCooperativeKernel((void*)dawn_nearfar<V, EI>, dim3(s->nf_grid), dim3(NT), args, 0, stream));
      return DAWN_OK;
    }
    KParams<V, EI> P = params(s, max_rounds);
    void* args[] = {&P};
    void* fn = kernel_for(s, P.pred_on != 0);
    CK(cudaLaunchCooperativeKernel(fn, dim3(P.pred_on ? s->grid_pred : s->grid), dim3(NT), args, s->smem,
                                   stream));
    // the worklist tail, when the persistent kernel handed over (it returns at once otherwise)
    if (P.wl_ring && P.live && P.algo == 0 && max_rounds == 0xFFFFFFFFu && !s->g->has_negative && !s->fb) {
      dawn_worklist<V, EI><<<s->wl_grid, NT, 0, stream>>>(P);
      CK(cudaGetLastError());
    }
    return DAWN_OK;
  }

  static int decode(dawn_solver_t s, double* dist_out, int64_t* pred_out, cudaStream_t stream) {
    const int64_t n = s->g->n;
    const int blocks = (int)std::min<int64_t>(148 * 16, (n + 255) / 256);
    if (dist_out) {
      const bool dev = is_device_ptr(dist_out);
      double* target = dev ? dist_out : s->dbuf;
      if (s->g->has_negative) dawn_decode_dist<V, false><<<blocks, 256, 0, stream>>>((const K*)s->dist, (uint32_t)n, target);
      else dawn_decode_dist<V, true><<<blocks, 256, 0, stream>>>((const K*)s->dist, (uint32_t)n, target);
      CK(cudaGetLastError());
      if (!dev) CK(cudaMemcpyAsync(dist_out, s->dbuf, 8 * (size_t)n, cudaMemcpyDeviceToHost, stream));
    }
    if (pred_out) {
      if (!s->pred) return fail(DAWN_EINVAL, "solver was created without DAWN_F_PRED");
      const bool dev = is_device_ptr(pred_out);
      int64_t* target = dev ? pred_out : s->pbuf;
      dawn_decode_pred<V><<<blocks, 256, 0, stream>>>((const K*)s->dist, s->pred, (uint32_t)n,
                                                      (uint32_t)s->source, target);
      CK(cudaGetLastError());
      if (!dev) CK(cudaMemcpyAsync(pred_out, s->pbuf, 8 * (size_t)n, cudaMemcpyDeviceToHost, stream));
    }
    return DAWN_OK;
  }


  // ---------------- batched multi-source (dawn_batch.cuh) ----------------
  static int batch_alloc(dawn_solver_t s) {
    if (s->batch_ready) return DAWN_OK;
    const int64_t n = s->g->n, m = s->g->m;
    const size_t ks = sizeof(K), es = sizeof(EI);
    CK(dmalloc(&s->bd, ks * BL * (size_t)n));
    for (int i = 0; i < 4; ++i) CK(dmalloc(&s->bmask[i], 4 * (size_t)n));
    for (int q = 0; q < 2; ++q) {
      CK(dmalloc(&s->bqnode[q], 4 * (size_t)n));
      CK(dmalloc(&s->bqmask[q], 4 * (size_t)n));
      CK(dmalloc(&s->bqoff[q], es * (size_t)n));
      CK(dmalloc(&s->bqbase[q], es * (size_t)n));
      CK(dmalloc(&s->btile[q], 4 * (size_t)(m / BWT + 4)));
    }
    CK(dmalloc(&s->bqkey, ks * BL * (size_t)n));
    CK(dmalloc(&s->bst, sizeof(BState)));
    CK(cudaMemset(s->bst, 0, sizeof(BState)));
    CK(cudaMemset(s->bmask[0], 0, 4 * (size_t)n));
    auto k = dawn_batch_persistent<V, EI, false>;
    auto kl = dawn_batch_persistent<V, EI, true>;  // async schedule (live distance lines)
    const size_t sm = sizeof(BSmem<V, EI>);
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    {
      const double need_kb = DAWN_BATCH_MIN_BLOCKS * ((double)(sm + 8 * 1024) / 1024.0 + 1.0);
      const int pct = std::min(100, (int)std::ceil(100.0 * need_kb / 228.0));
      CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
      CK(cudaFuncSetAttribute(kl, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    }
    int bps = 0, nsm = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int bpl = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, NT, sm));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpl, kl, NT, sm));
    bps = std::min(bps, bpl);  // one grid size for both instances
    if (bps < 1) return fail(DAWN_ECUDA, "batched kernel cannot be resident");
    const int64_t work = std::max<int64_t>((n + TILE - 1) / TILE, (m + BWT * WPB - 1) / (BWT * WPB));
    s->bgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)bps * nsm, work));
    s->bsmem = sm;
    s->batch_ready = true;
    return DAWN_OK;
  }

  static BParams<V, EI> bparams(dawn_solver_t s, const int64_t* src, int nl, int algo) {
    dawn_graph_t g = s->g;
    BParams<V, EI> P;
    P.n = (uint32_t)g->n;
    P.nlanes = (uint32_t)nl;
    P.row_ptr = (const EI*)g->row_ptr;
    P.e2 = g->e2;
    P.ecol = g->ecol;
    P.ew = g->ew;
    P.bd = (K*)s->bd;
    P.nmask = s->bmask[0];
    P.w1 = s->bmask[1];
    P.w2 = s->bmask[2];
    P.smask = s->bmask[3];
    for (int q = 0; q < 2; ++q) {
      P.qnode[q] = s->bqnode[q];
      P.qmask[q] = s->bqmask[q];
      P.qoff[q] = (EI*)s->bqoff[q];
      P.qbase[q] = (EI*)s->bqbase[q];
      P.tile_row[q] = s->btile[q];
    }
    P.qkey = (K*)s->bqkey;
    P.st = s->bst;
    for (int l = 0; l < BL; ++l) P.src[l] = l < nl ? (uint32_t)src[l] : 0xFFFFFFFFu;
    P.ebits = s->ebits;
    P.algo = algo;
    P.sparse_util = (uint32_t)s->batch_sparse_util;
    P.prof = s->prof;
    P.prof_cap = s->prof_cap;
    return P;
  }

  // one batch of nl <= 32 sources; nmask is all-zero on entry and on exit
  static int batch_run(dawn_solver_t s, const int64_t* src, int nl, int algo, bool live, cudaStream_t stream) {
    TRY(batch_alloc(s));
    const int64_t n = s->g->n;
    CK(cudaMemsetAsync(s->bd, 0xFF, sizeof(K) * BL * (size_t)n, stream));
    CK(cudaMemsetAsync(s->bmask[1], 0, 4 * (size_t)n, stream));
    CK(cudaMemsetAsync(s->bmask[2], 0, 4 * (size_t)n, stream));
    CK(cudaMemsetAsync(s->bmask[3], 0, 4 * (size_t)n, stream));
    if (s->prof) CK(cudaMemsetAsync(s->prof, 0, 32 * (size_t)s->prof_cap, stream));
    BParams<V, EI> P = bparams(s, src, nl, algo);
    dawn_batch_init<V, EI><<<1, 32, 0, stream>>>(P);
    CK(cudaGetLastError());
    void* args[] = {&P};
    CK(cudaLaunchCooperativeKernel(live ? (void*)dawn_batch_persistent<V, EI, true> : (void*)dawn_batch_persistent<V, EI, false>,
                                   dim3(s->bgrid), dim3(NT), args, s->bsmem,
                                   stream));
    return DAWN_OK;
  }

  // decode the batch into rows [nl][ld] of double (out_vt F64) or the value type (F32 graphs)
  static int batch_decode(dawn_solver_t s, void* out, int out_vt, int64_t ld, int nl, cudaStream_t stream) {
    const int64_t n = s->g->n;
    const int blocks = (int)std::min<int64_t>(148 * 8, (n + 31) / 32);
    const bool dev = is_device_ptr(out);
    const size_t es = out_vt == DAWN_F64 ? 8 : 4;
    void* target = out;
    if (!dev) {
      if (!s->bout) CK(dmalloc(&s->bout, 8 * BL * (size_t)n));
      target = s->bout;
    }
    const int64_t tld = dev ? ld : n;
    if (out_vt == DAWN_F64)
      dawn_batch_decode<V, double><<<blocks, 256, 0, stream>>>((const K*)s->bd, (uint32_t)n, (uint32_t)nl,
                                                               (double*)target, (size_t)tld);
    else
      dawn_batch_decode<V, float><<<blocks, 256, 0, stream>>>((const K*)s->bd, (uint32_t)n, (uint32_t)nl,
                                                              (float*)target, (size_t)tld);
    CK(cudaGetLastError());
    if (!dev)
      CK(cudaMemcpy2DAsync(out, es * (size_t)ld, target, es * (size_t)n, es * (size_t)n, (size_t)nl,
                           cudaMemcpyDeviceToHost, stream));
    return DAWN_OK;
  }

  static int alloc(dawn_solver_t s) {
    const int64_t n = s->g->n, m = s->g->m;
    const size_t ks = sizeof(K), es = sizeof(EI);
    CK(dmalloc(&s->dist, ks * n));
    CK(dmalloc(&s->stamp, 4 * n));
    CK(dmalloc(&s->phist, 4 * 2 * PW_BINS));
    CK(cudaMemset(s->phist, 0, 4 * 2 * PW_BINS));
    CK(dmalloc(&s->bmap, 4 * (size_t)((n + 31) / 32 + 4)));  // padded for 16-byte loads
    CK(dmalloc(&s->wstate, (size_t)n + 4));  // + 4: the worklist tail updates it by 32-bit words
    if (!s->g->has_negative) {
      // worklist tail (async schedule): ring of items (every node once + long-row chunks + slack;
      // a full ring only makes producers wait)
      const uint64_t need = (uint64_t)n + (uint64_t)(m / WT_MIN) + (1ull << 16);
      uint64_t cap = 1;
      while (cap < need) cap <<= 1;
      s->wl_cap = cap;
      CK(dmalloc(&s->wl_ring, 16 * cap));  // 16-byte items; node field 0xFFFFFFFF = empty
      CK(cudaMemset(s->wl_ring, 0xFF, 16 * cap));
    }
    if (s->flags & (DAWN_F_PRED | DAWN_F_NEGCHECK)) {
      CK(dmalloc(&s->pred, 8 * n));
      CK(dmalloc(&s->jmp0, 4 * n));
      CK(dmalloc(&s->jmp1, 4 * n));
      CK(dmalloc(&s->pbuf, 8 * n));
    }
    for (int i = 0; i < 2; ++i) {
      CK(dmalloc(&s->qnode[i], 4 * n));
      CK(dmalloc(&s->qoff[i], es * n));
      CK(dmalloc(&s->qbase[i], es * n));
      CK(dmalloc(&s->qkey[i], ks * n));
    }
    CK(dmalloc(&s->tile_row, 4 * (size_t)(m / WT_MIN + 4)));
    CK(dmalloc(&s->st, sizeof(DevState)));
    CK(cudaMemset(s->st, 0, sizeof(DevState)));
    CK(hmalloc(&s->st_host, sizeof(DevState)));
    CK(dmalloc(&s->dbuf, 8 * n));
    if (s->flags & DAWN_F_PROFILE) {
      s->prof_cap = 1u << 16;
      CK(dmalloc(&s->prof, 32 * (size_t)s->prof_cap));
      CK(dmalloc(&s->cta_prof, 8 * 2 * 2048 * (size_t)CTA_PROF_ROUNDS));
      CK(cudaMemset(s->cta_prof, 0, 8 * 2 * 2048 * (size_t)CTA_PROF_ROUNDS));
    }
    return setup(s);
  }
};

#define DISPATCH(g, CALL)                                                         \
  ([&]() -> int {                                                                 \
    switch ((g)->vtype) {                                                         \
      case DAWN_I32:                                                              \
        return (g)->wide ? Impl<int32_t, unsigned long long>::CALL : Impl<int32_t, uint32_t>::CALL; \
      case DAWN_I64:                                                              \
        return (g)->wide ? Impl<int64_t, unsigned long long>::CALL : Impl<int64_t, uint32_t>::CALL; \
      case DAWN_F32:                                                              \
        return (g)->wide ? Impl<float, unsigned long long>::CALL : Impl<float, uint32_t>::CALL;     \
      default:                                                                    \
        return (g)->wide ? Impl<double, unsigned long long>::CALL : Impl<double, uint32_t>::CALL;   \
    }                                                                             \
  }())

static void solver_free(dawn_solver_t s) {
  if (!s) return;
  cudaSetDevice(s->g->device);
  cudaDeviceSynchronize();
  dfree(s->dist);
  dfree(s->stamp);
  dfree(s->phist);
  dfree(s->bmap);
  dfree(s->wstate);
  dfree(s->pred);
  dfree(s->jmp0);
  dfree(s->jmp1);
  dfree(s->pbuf);
  for (int i = 0; i < 2; ++i) {
    dfree(s->qnode[i]);
    dfree(s->qoff[i]);
    dfree(s->qbase[i]);
    dfree(s->qkey[i]);
  }
  dfree(s->tile_row);
  dfree(s->wl_ring);
  dfree(s->st);
  hfree(s->st_host);
  dfree(s->dbuf);
  dfree(s->prof);
  dfree(s->cta_prof);
  dfree(s->bd);
  for (int i = 0; i < 4; ++i) dfree(s->bmask[i]);
  for (int q = 0; q < 2; ++q) {
    dfree(s->bqnode[q]);
    dfree(s->bqmask[q]);
    dfree(s->bqoff[q]);
    dfree(s->bqbase[q]);
    dfree(s->btile[q]);
  }
  dfree(s->bqkey);
  dfree(s->bst);
  hfree(s->bst_host);
  dfree(s->bout);
  delete s;
}

extern "C" int dawn_solver_create(dawn_graph_t g, unsigned flags, dawn_solver_t* out) {
  if (!g || !out) return fail(DAWN_EINVAL, "NULL argument");
  *out = nullptr;
  CK(cudaSetDevice(g->device));
  dawn_solver_s* s = new dawn_solver_s();
  s->g = g;
  s->flags = flags;
  s->ebits = 64 - bitlen((uint64_t)g->n);
  int lg = 0;
  while ((1ll << lg) < g->n) ++lg;
  s->logn = lg;
  int rc = DISPATCH(g, alloc(s));
  if (rc != DAWN_OK) {
    solver_free(s);
    return rc;
  }
  *out = s;
  return DAWN_OK;
}

extern "C" int dawn_solver_tune(dawn_solver_t s, const char* key, double value) {
  if (!s || !key) return fail(DAWN_EINVAL, "NULL argument");
  if (!strcmp(key, "dense_edges_per_node")) {
    if (!(value >= 0.0)) return fail(DAWN_EINVAL, "dense_edges_per_node must be >= 0");
    s->dense_edges_per_node = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "worklist_edges")) {
    if (!(value >= 0.0)) return fail(DAWN_EINVAL, "worklist_edges must be >= 0");
    s->worklist_edges = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "wide_tiles")) {
    if (!(value == -1.0 || value == 0.0 || value == 1.0)) return fail(DAWN_EINVAL, "wide_tiles must be -1, 0 or 1");
    s->wide_pref = (int)value;
    CK(cudaSetDevice(s->g->device));
    return DISPATCH(s->g, setup(s));
  }
  if (!strcmp(key, "bitmap_frontier")) {
    if (!(value == -1.0 || value == 0.0 || value == 1.0)) return fail(DAWN_EINVAL, "bitmap_frontier must be -1, 0 or 1");
    s->fb_pref = (int)value;
    CK(cudaSetDevice(s->g->device));
    return DISPATCH(s->g, setup(s));
  }
  if (!strcmp(key, "nearfar")) {
    if (!(value == -1.0 || value == 0.0 || value == 1.0)) return fail(DAWN_EINVAL, "nearfar must be -1, 0 or 1");
    s->nf_pref = (int)value;
    CK(cudaSetDevice(s->g->device));
    return DISPATCH(s->g, setup(s));
  }
  if (!strcmp(key, "small_graph")) {
    if (!(value == -1.0 || value == 0.0 || value == 1.0)) return fail(DAWN_EINVAL, "small_graph must be -1, 0 or 1");
    s->small_pref = (int)value;
    CK(cudaSetDevice(s->g->device));
    return DISPATCH(s->g, setup(s));
  }
  if (!strcmp(key, "speculate_negcheck")) {
    if (!(value == 0.0 || value == 1.0)) return fail(DAWN_EINVAL, "speculate_negcheck must be 0 or 1");
    s->spec = value != 0.0;
    return DAWN_OK;
  }
  if (!strcmp(key, "small_cluster")) {
    if (!(value == 1.0 || value == 2.0 || value == 4.0 || value == 8.0 || value == 16.0))
      return fail(DAWN_EINVAL, "small_cluster must be 1, 2, 4, 8 or 16");
    s->small_cl_max = (int)value;
    CK(cudaSetDevice(s->g->device));
    return DISPATCH(s->g, setup(s));
  }
  if (!strcmp(key, "nearfar_delta")) {
    if (!(value >= 0.0)) return fail(DAWN_EINVAL, "nearfar_delta must be >= 0");
    s->nf_delta = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "nearfar_batches")) {
    if (!(value >= 0.0)) return fail(DAWN_EINVAL, "nearfar_batches must be >= 0");
    s->nf_cap = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "priority_frac")) {
    if (!(value >= 0.0 && value <= 1.0)) return fail(DAWN_EINVAL, "priority_frac must be in [0, 1]");
    s->pw_frac = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "priority_edges_per_edge")) {
    if (!(value >= 0.0)) return fail(DAWN_EINVAL, "priority_edges_per_edge must be >= 0");
    s->pw_edges_per_edge = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "priority_seed_edges")) {
    if (!(value >= 0.0)) return fail(DAWN_EINVAL, "priority_seed_edges must be >= 0");
    s->pw_seed_edges = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "nearfar_delta_mean")) {
    if (!(value > 0.0)) return fail(DAWN_EINVAL, "nearfar_delta_mean must be > 0");
    s->nf_delta_mean = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "batch_sparse_util")) {
    if (!(value >= 0.0 && value <= 33.0)) return fail(DAWN_EINVAL, "batch_sparse_util must be in [0, 33]");
    s->batch_sparse_util = value;
    return DAWN_OK;
  }
  if (!strcmp(key, "batch_min_sources")) {
    if (!(value >= 0.0)) return fail(DAWN_EINVAL, "batch_min_sources must be >= 0");
    s->batch_min_sources = value;
    return DAWN_OK;
  }
  return fail(DAWN_EINVAL, "unknown tuning key '%s'", key);
}

extern "C" int dawn_solver_destroy(dawn_solver_t s) {
  solver_free(s);
  return DAWN_OK;
}

static int check_solve_args(dawn_solver_t s, int64_t source, int algo, unsigned flags) {
  if (!s) return fail(DAWN_EINVAL, "solver is NULL");
  if (source < 0 || source >= s->g->n)
    return fail(DAWN_ESOURCE, "source %lld out of range for n=%lld", (long long)source, (long long)s->g->n);
  if (algo != DAWN_GOVM && algo != DAWN_GSVM) return fail(DAWN_EINVAL, "unknown algo %d", algo);
  if ((flags & DAWN_F_PRED) && !(s->flags & DAWN_F_PRED))
    return fail(DAWN_EINVAL, "DAWN_F_PRED requested but the solver was created without it");
  return DAWN_OK;
}

static int do_begin(dawn_solver_t s, int64_t source, int algo, unsigned flags, cudaStream_t st) {
  CK(cudaSetDevice(s->g->device));
  s->source = source;
  s->algo = algo;
  s->last_batch = false;
  s->run_flags = flags & (s->flags | DAWN_F_NEGCHECK | DAWN_F_ASYNC);
  if ((s->run_flags & DAWN_F_NEGCHECK) && !s->pred) s->run_flags &= ~DAWN_F_NEGCHECK;
  s->active = true;
  return DISPATCH(s->g, begin(s, st));
}

static void fill_stats(const DevState& d, dawn_stats_t* o) {
  o->outer_steps = (int64_t)d.steps;
  o->relaxations = (int64_t)d.R;
  o->writes = (int64_t)d.W;
  o->first_discoveries = (int64_t)d.FD;
  o->multi_written = (int64_t)d.multi;
  o->negative_cycle = d.flag ? 1 : 0;
  o->early_exit = d.early ? 1 : 0;
}

static int read_state(dawn_solver_t s, cudaStream_t st) {
  CK(cudaMemcpyAsync(s->st_host, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (s->st_host->abort)
    return fail(DAWN_ECUDA, "device watchdog: the solve made no progress for 30 s and was aborted");
  return DAWN_OK;
}

extern "C" int dawn_sssp(dawn_solver_t s, int64_t source, int algo, unsigned flags,
                         double* dist_out, int64_t* pred_out, dawn_stats_t* stats_out,
                         void* stream) {
  TRY(check_solve_args(s, source, algo, flags));
  if (pred_out && !(flags & DAWN_F_PRED)) return fail(DAWN_EINVAL, "pred_out requires DAWN_F_PRED");
  cudaStream_t st = (cudaStream_t)stream;
  TRY(do_begin(s, source, algo, flags, st));
  TRY(DISPATCH(s->g, run(s, 0xFFFFFFFFu, st)));
  TRY(DISPATCH(s->g, decode(s, dist_out, pred_out, st)));
  if (stats_out) {
    TRY(read_state(s, st));
    fill_stats(*s->st_host, stats_out);
  }
  return DAWN_OK;
}

extern "C" int dawn_sssp_begin(dawn_solver_t s, int64_t source, int algo, unsigned flags,
                               void* stream) {
  TRY(check_solve_args(s, source, algo, flags));
  return do_begin(s, source, algo, flags, (cudaStream_t)stream);
}

extern "C" int dawn_sssp_advance(dawn_solver_t s, int max_rounds, int64_t* round_out,
                                 int* done_out, void* stream) {
  if (!s || !s->active) return fail(DAWN_EINVAL, "no active solve");
  if (max_rounds < 1) return fail(DAWN_EINVAL, "max_rounds must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  if (s->init_pending) TRY(DISPATCH(s->g, init_solve(s, st)));
  TRY(read_state(s, st));
  if (!s->st_host->done) {
    TRY(DISPATCH(s->g, run(s, (unsigned)max_rounds, st)));
    TRY(read_state(s, st));
  }
  if (round_out) *round_out = (int64_t)s->st_host->round - 1;
  if (done_out) *done_out = s->st_host->done ? 1 : 0;
  return DAWN_OK;
}

extern "C" int dawn_sssp_run(dawn_solver_t s, int max_rounds, void* stream) {
  if (!s || !s->active) return fail(DAWN_EINVAL, "no active solve");
  if (max_rounds < 0) return fail(DAWN_EINVAL, "max_rounds must be >= 0");
  CK(cudaSetDevice(s->g->device));
  return DISPATCH(s->g, run(s, max_rounds == 0 ? 0xFFFFFFFFu : (unsigned)max_rounds, (cudaStream_t)stream));
}

extern "C" int dawn_solver_state(dawn_solver_t s, double* dist_out, uint32_t* stamp_out,
                                 void* stream) {
  if (!s || !s->active) return fail(DAWN_EINVAL, "no active solve");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  if (s->init_pending) TRY(DISPATCH(s->g, init_solve(s, st)));
  TRY(DISPATCH(s->g, decode(s, dist_out, nullptr, st)));
  if (stamp_out)
    CK(cudaMemcpyAsync(stamp_out, s->stamp, 4 * (size_t)s->g->n, cudaMemcpyDefault, st));
  CK(cudaStreamSynchronize(st));
  return DAWN_OK;
}

extern "C" int dawn_solver_result(dawn_solver_t s, double* dist_out, int64_t* pred_out,
                                  dawn_stats_t* stats_out, void* stream) {
  if (!s || !s->active) return fail(DAWN_EINVAL, "no solve has run on this solver");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  if (pred_out && !(s->run_flags & DAWN_F_PRED)) return fail(DAWN_EINVAL, "last solve did not record predecessors");
  if (s->init_pending) TRY(DISPATCH(s->g, init_solve(s, st)));
  TRY(DISPATCH(s->g, decode(s, dist_out, pred_out, st)));
  TRY(read_state(s, st));
  if (stats_out) fill_stats(*s->st_host, stats_out);
  return DAWN_OK;
}

extern "C" int dawn_solver_round_profile(dawn_solver_t s, uint64_t* out, int64_t cap_rounds,
                                         int64_t* nrounds, void* stream) {
  if (!s || !(s->active || s->last_batch)) return fail(DAWN_EINVAL, "no solve has run on this solver");
  if (!s->prof) return fail(DAWN_EINVAL, "solver was created without DAWN_F_PROFILE");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  int64_t rounds_run = 0;
  if (s->last_batch) {
    BState b;
    CK(cudaMemcpyAsync(&b, s->bst, sizeof(BState), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    rounds_run = (int64_t)b.rounds + 2;
  } else {
    TRY(read_state(s, st));
    rounds_run = (int64_t)s->st_host->round;
  }
  const int64_t done = std::min<int64_t>(rounds_run, (int64_t)s->prof_cap);
  const int64_t k = std::min<int64_t>(done, cap_rounds);
  if (out && k > 0) CK(cudaMemcpy(out, s->prof, 32 * (size_t)k, cudaMemcpyDeviceToHost));
  if (nrounds) *nrounds = done;
  return DAWN_OK;
}

extern "C" int dawn_solver_cta_profile(dawn_solver_t s, uint64_t* out, int64_t cap_rounds, int* grid_out,
                                       void* stream) {
  if (!s || !s->cta_prof) return fail(DAWN_EINVAL, "solver was created without DAWN_F_PROFILE");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  CK(cudaStreamSynchronize(st));
  const int64_t k = std::min<int64_t>(cap_rounds, (int64_t)CTA_PROF_ROUNDS);
  if (grid_out) *grid_out = s->grid;
#ifdef DAWN_XTIMING  // debug variant: the per-warp X-phase checkpoints [16][2368][6]
  if (out) CK(cudaMemcpy(out, s->cta_prof, 8 * (size_t)16 * 2368 * 6, cudaMemcpyDeviceToHost));
  (void)k;
#else
  if (out && k > 0) CK(cudaMemcpy(out, s->cta_prof, 8 * 2 * (size_t)s->grid * (size_t)k, cudaMemcpyDeviceToHost));
#endif
  return DAWN_OK;
}

extern "C" int dawn_solver_worklist_stats(dawn_solver_t s, uint64_t* out, void* stream) {
  if (!s || !out) return fail(DAWN_EINVAL, "NULL argument");
  if (!s->active) return fail(DAWN_EINVAL, "no active solve");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  TRY(read_state(s, st));
  const DevState& d = *s->st_host;
  const bool ran = d.wl_mode != 0u;
  out[0] = ran ? d.steps : 0;
  out[1] = ran ? d.wl_items : 0;
  out[2] = ran ? d.wl_batches : 0;
  out[3] = ran ? d.wl_busy_ns : 0;
  out[4] = ran ? d.wl_wait_ns : 0;
  out[5] = (ran && d.wl_t1 > d.wl_t0) ? d.wl_t1 - d.wl_t0 : 0;
  return DAWN_OK;
}

static bool batch_ok(dawn_solver_t s, int algo, unsigned flags) {
  return !s->g->has_negative && s->g->n >= 2 && !(flags & DAWN_F_PRED) && (algo == DAWN_GOVM || algo == DAWN_GSVM);
}

extern "C" int dawn_batch_supported(dawn_solver_t s, int algo, unsigned flags, int* out) {
  if (!s || !out) return fail(DAWN_EINVAL, "NULL argument");
  *out = batch_ok(s, algo, flags) ? 1 : 0;
  return DAWN_OK;
}

static void fill_batch_stats(const BState& b, int nl, int64_t n, dawn_stats_t* o) {
  for (int l = 0; l < nl; ++l) {
    const int64_t lw = (int64_t)b.lastw[l];
    o[l].outer_steps = std::min<int64_t>(std::max<int64_t>(lw + 1, 2), n);
    o[l].relaxations = (int64_t)b.R[l];
    o[l].writes = (int64_t)b.W[l];
    o[l].first_discoveries = (int64_t)b.FD[l];
    o[l].multi_written = (int64_t)b.MW[l];
    o[l].negative_cycle = (((b.guard >> l) & 1u) || lw >= n) ? 1 : 0;
    o[l].early_exit = 0;
  }
}

extern "C" int dawn_mssp_batch(dawn_solver_t s, const int64_t* sources, int64_t k, int algo, unsigned flags,
                               void* dist_out, int out_vtype, int64_t ld, dawn_stats_t* stats_out, void* stream) {
  if (!s) return fail(DAWN_EINVAL, "solver is NULL");
  if (k < 0 || (k > 0 && !sources)) return fail(DAWN_EINVAL, "bad sources");
  for (int64_t i = 0; i < k; ++i) TRY(check_solve_args(s, sources[i], algo, flags & ~DAWN_F_PRED));
  if (!batch_ok(s, algo, flags))
    return fail(DAWN_EUNSUPPORTED, "batched solve needs non-negative weights, n >= 2 and no predecessors");
  if (dist_out) {
    if (out_vtype != DAWN_F64 && !(out_vtype == DAWN_F32 && s->g->vtype == DAWN_F32))
      return fail(DAWN_EINVAL, "out_vtype must be DAWN_F64 (or DAWN_F32 for a float32 graph)");
    if (ld < s->g->n) return fail(DAWN_EINVAL, "ld must be >= n");
  }
  if (k == 0) return DAWN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  const int64_t n = s->g->n;
  const int64_t nb = (k + BL - 1) / BL;
  if (stats_out && s->bst_host_cap < nb) {
    CK(cudaStreamSynchronize(st));  // a previous asynchronous call may still write the old buffer
    hfree(s->bst_host);
    s->bst_host = nullptr;
    s->bst_host_cap = 0;
    CK(hmalloc(&s->bst_host, sizeof(BState) * nb));
    s->bst_host_cap = nb;
  }
  const size_t es = out_vtype == DAWN_F64 ? 8 : 4;
  const bool host_out = dist_out && !is_device_ptr(dist_out);
  s->last_batch = true;
  for (int64_t b = 0; b < nb; ++b) {
    const int nl = (int)std::min<int64_t>(BL, k - b * BL);
    TRY(DISPATCH(s->g, batch_run(s, sources + b * BL, nl, algo, (flags & DAWN_F_ASYNC) != 0, st)));
    if (dist_out)
      TRY(DISPATCH(s->g, batch_decode(s, (char*)dist_out + (size_t)b * BL * ld * es, out_vtype, ld, nl, st)));
    if (stats_out) CK(cudaMemcpyAsync(s->bst_host + b, s->bst, sizeof(BState), cudaMemcpyDeviceToHost, st));
  }
  if (stats_out || host_out) {
    CK(cudaStreamSynchronize(st));
    if (stats_out)
      for (int64_t b = 0; b < nb; ++b) {
        if (s->bst_host[b].abort)
          return fail(DAWN_ECUDA, "device watchdog: a batch made no progress for 30 s and was aborted");
        fill_batch_stats(s->bst_host[b], (int)std::min<int64_t>(BL, k - b * BL), n, stats_out + b * BL);
      }
  }
  return DAWN_OK;
}

extern "C" int dawn_mssp(dawn_solver_t s, const int64_t* sources, int64_t k, int algo,
                         unsigned flags, double* dist_out, dawn_stats_t* stats_out, void* stream) {
  if (!s) return fail(DAWN_EINVAL, "solver is NULL");
  if (k < 0 || (k > 0 && !sources)) return fail(DAWN_EINVAL, "bad sources");
  for (int64_t i = 0; i < k; ++i) TRY(check_solve_args(s, sources[i], algo, flags & ~DAWN_F_PRED));
  if (k > 0 && (double)k >= s->batch_min_sources && batch_ok(s, algo, flags))
    return dawn_mssp_batch(s, sources, k, algo, flags, dist_out, DAWN_F64, s->g->n, stats_out, stream);
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(s->g->device));
  DevState* hs = nullptr;
  if (stats_out && k > 0) CK(hmalloc(&hs, sizeof(DevState) * k));
  const int64_t n = s->g->n;
  int rc = DAWN_OK;
  for (int64_t i = 0; i < k && rc == DAWN_OK; ++i) {
    rc = do_begin(s, sources[i], algo, flags & ~DAWN_F_PRED, st);
    if (rc == DAWN_OK) rc = DISPATCH(s->g, run(s, 0xFFFFFFFFu, st));
    if (rc == DAWN_OK && dist_out) rc = DISPATCH(s->g, decode(s, dist_out + i * n, nullptr, st));
    if (rc == DAWN_OK && hs) {
      cudaError_t e = cudaMemcpyAsync(hs + i, s->st, sizeof(DevState), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) rc = fail(DAWN_ECUDA, "stats copy: %s", cudaGetErrorString(e));
    }
  }
  if (rc == DAWN_OK) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(DAWN_ECUDA, "mssp: %s", cudaGetErrorString(e));
  }
  if (rc == DAWN_OK && hs)
    for (int64_t i = 0; i < k && rc == DAWN_OK; ++i) {
      if (hs[i].abort) rc = fail(DAWN_ECUDA, "device watchdog: a solve made no progress for 30 s and was aborted");
      else fill_stats(hs[i], stats_out + i);
    }
  if (hs) hfree(hs);
  return rc;
}

// ---------------------------------------------------------------------------
// canonical CSR construction (build_csr, graph.py:303-322) on the device
// ---------------------------------------------------------------------------
static int bits_for(unsigned long long x) {
  int b = 0;
  while (b < 64 && (x >> b) != 0ull) ++b;
  return b;
}

extern "C" int dawn_build_csr(int device, int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                              const double* w, int src_is_device, int64_t* row_ptr_out, int64_t* col_out,
                              double* val_out, void* stream) {
  if (n < 0 || m < 0 || !row_ptr_out || (m > 0 && (!u || !v || !w || !col_out || !val_out)))
    return fail(DAWN_EINVAL, "bad build_csr arguments (n=%lld, m=%lld)", (long long)n, (long long)m);
  if (n > 0 && (unsigned long long)n > 0xFFFFFFFFull)
    return fail(DAWN_EUNSUPPORTED, "n=%lld exceeds the 2^32 node limit of the 64-bit sort key", (long long)n);
  CK(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  const bool out_dev = is_device_ptr(row_ptr_out);
  const int blocks = 148 * 8;
  if (m == 0) {
    if (out_dev) {
      k_csr_empty<<<blocks, 256, 0, st>>>(n, row_ptr_out);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(st));
    } else {
      memset(row_ptr_out, 0, 8 * (size_t)(n + 1));
    }
    return DAWN_OK;
  }
  // device workspace: staged inputs (host sources), keys/idx in and out, outputs, temp storage
  size_t tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const unsigned long long*)nullptr,
                                     (unsigned long long*)nullptr, (const unsigned long long*)nullptr,
                                     (unsigned long long*)nullptr, m, 0, 64, st));
  const size_t in_bytes = src_is_device ? 0 : 24 * (size_t)m;
  const size_t out_bytes = out_dev ? 0 : 8 * (size_t)(n + 1) + 16 * (size_t)m;
  const size_t total = in_bytes + 32 * (size_t)m + out_bytes + tmp_bytes + 64;
  char* ws = nullptr;
  CK(dmalloc(&ws, total));
  auto release = [&](int rc) {
    cudaStreamSynchronize(st);
    dfree(ws);
    return rc;
  };
  char* q = ws;
  const int64_t* du = u;
  const int64_t* dv = v;
  const double* dw = w;
  cudaError_t e;
  if (!src_is_device) {
    int64_t* su = (int64_t*)q;
    int64_t* sv = su + m;
    double* sw = (double*)(sv + m);
    q += in_bytes;
    if ((e = cudaMemcpyAsync(su, u, 8 * (size_t)m, cudaMemcpyDefault, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(sv, v, 8 * (size_t)m, cudaMemcpyDefault, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(sw, w, 8 * (size_t)m, cudaMemcpyDefault, st)) != cudaSuccess)
      return release(fail(DAWN_ECUDA, "edge upload: %s", cudaGetErrorString(e)));
    du = su;
    dv = sv;
    dw = sw;
  }
  unsigned long long* k0 = (unsigned long long*)q;
  unsigned long long* k1 = k0 + m;
  unsigned long long* i0 = k1 + m;
  unsigned long long* i1 = i0 + m;
  q += 32 * (size_t)m;
  int64_t* rp = row_ptr_out;
  int64_t* col = col_out;
  double* val = val_out;
  if (!out_dev) {
    rp = (int64_t*)q;
    col = rp + (n + 1);
    val = (double*)(col + m);
    q += out_bytes;
  }
  void* tmp = q;
  q += tmp_bytes;
  unsigned* flags = (unsigned*)(((uintptr_t)q + 15) & ~(uintptr_t)15);
  if ((e = cudaMemsetAsync(flags, 0, sizeof(unsigned), st)) != cudaSuccess)
    return release(fail(DAWN_ECUDA, "flags: %s", cudaGetErrorString(e)));
  k_csr_keys<<<blocks, 256, 0, st>>>(du, dv, dw, n, m, k0, i0, flags);
  if ((e = cudaGetLastError()) != cudaSuccess) return release(fail(DAWN_ECUDA, "keys: %s", cudaGetErrorString(e)));
  const int kbits = std::max(1, bits_for((unsigned long long)n * (unsigned long long)n - 1ull));
  if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i0, i1, m, 0, kbits, st)) != cudaSuccess)
    return release(fail(DAWN_ECUDA, "sort: %s", cudaGetErrorString(e)));
  k_csr_emit<<<blocks, 256, 0, st>>>(k1, i1, dw, n, m, col, val);
  k_csr_rowptr<<<blocks, 256, 0, st>>>(k1, n, m, rp);
  if ((e = cudaGetLastError()) != cudaSuccess) return release(fail(DAWN_ECUDA, "emit: %s", cudaGetErrorString(e)));
  unsigned hflags = 0;
  if ((e = cudaMemcpyAsync(&hflags, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return release(fail(DAWN_ECUDA, "build_csr: %s", cudaGetErrorString(e)));
  if (hflags & CSR_ERR_NODE) return release(fail(DAWN_EINVAL, "edge endpoint out of range for n=%lld", (long long)n));
  if (hflags & CSR_ERR_WEIGHT) return release(fail(DAWN_EINVAL, "non-finite edge weight"));
  if (!out_dev) {
    if ((e = cudaMemcpyAsync(row_ptr_out, rp, 8 * (size_t)(n + 1), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(col_out, col, 8 * (size_t)m, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(val_out, val, 8 * (size_t)m, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      return release(fail(DAWN_ECUDA, "csr download: %s", cudaGetErrorString(e)));
  }
  return release(DAWN_OK);
}

// ---------------------------------------------------------------------------
// synthetic RMAT generator (counter-based, see generators.py for the spec)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long draw64(unsigned long long seed, unsigned long long i,
                                                     unsigned lvl) {
  return mix64(seed * 0x9E3779B97F4A7C15ull + i * 64ull + lvl + 0x9E3779B97F4A7C15ull);
}

__global__ void k_gen_rmat(int scale, int64_t m, uint32_t A, uint32_t AB, uint32_t ABC,
                           unsigned long long seed, int wkind, int64_t wlo, unsigned long long wrange,
                           unsigned long long wseed, int64_t* u_out, int64_t* v_out, double* w_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      const uint32_t q = (uint32_t)(draw64(seed, (unsigned long long)i, l) >> 40);
      const int ub = q >= AB;
      const int vb = (q >= A && q < AB) || q >= ABC;
      u |= (int64_t)ub << l;
      v |= (int64_t)vb << l;
    }
    const unsigned long long h = draw64(wseed, (unsigned long long)i, 63);
    double w;
    if (wkind == 0) w = (double)(wlo + (int64_t)(((h >> 32) * wrange) >> 32));
    else w = (double)((float)(h >> 40) * (1.0f / 16777216.0f));
    u_out[i] = u;
    v_out[i] = v;
    w_out[i] = w;
  }
}

extern "C" int dawn_gen_rmat(int device, int scale, int64_t edge_factor, double a, double b,
                             double c, uint64_t seed, int wkind, int64_t wlo, int64_t whi,
                             uint64_t wseed, int64_t* u_out, int64_t* v_out, double* w_out,
                             void* stream) {
  if (scale < 1 || scale > 31 || edge_factor < 1 || !u_out || !v_out || !w_out)
    return fail(DAWN_EINVAL, "bad rmat arguments");
  if (wkind == 0 && (whi < wlo || whi - wlo >= (1ll << 32))) return fail(DAWN_EINVAL, "bad weight range");
  CK(cudaSetDevice(device));
  const int64_t m = edge_factor << scale;
  const uint32_t A = (uint32_t)(a * 16777216.0), AB = (uint32_t)((a + b) * 16777216.0),
                 ABC = (uint32_t)((a + b + c) * 16777216.0);
  k_gen_rmat<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(scale, m, A, AB, ABC, seed, wkind, wlo,
                                                        (unsigned long long)(whi - wlo + 1), wseed,
                                                        u_out, v_out, w_out);
  CK(cudaGetLastError());
  return DAWN_OK;
}

// 4-neighbour grid written straight into CSR (grid_graph, generators.py:96-113).
// Row offsets are closed-form: a node in grid row i loses one edge per border
// it touches, so rows before i hold i(4C-2) - C[i>0] edges and the nodes
// before column j of row i hold j(4 - t_i) - [j>0], t_i = [i==0] + [i==R-1].
// Neighbours in ascending id (up, left, right, down); the weight of the edge
// at CSR position e is the same counter draw as the RMAT weights.
__global__ void k_gen_grid(int64_t R, int64_t C, int wkind, int64_t wlo, unsigned long long wrange,
                           unsigned long long wseed, int64_t* row_ptr, int64_t* col, double* val) {
  const int64_t n = R * C;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id <= n;
       id += (int64_t)gridDim.x * blockDim.x) {
    if (id == n) {
      row_ptr[n] = 4 * R * C - 2 * R - 2 * C;
      continue;
    }
    const int64_t i = id / C, j = id - i * C;
    const int64_t t = (i == 0) + (i == R - 1);
    int64_t e = i * (4 * C - 2) - (i > 0 ? C : 0) + j * (4 - t) - (j > 0);
    row_ptr[id] = e;
    const int64_t nb[4] = {i > 0 ? id - C : -1, j > 0 ? id - 1 : -1, j + 1 < C ? id + 1 : -1,
                           i + 1 < R ? id + C : -1};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (nb[k] < 0) continue;
      const unsigned long long h = draw64(wseed, (unsigned long long)e, 63);
      col[e] = nb[k];
      val[e] = wkind == 0 ? (double)(wlo + (int64_t)(((h >> 32) * wrange) >> 32))
                          : (double)((float)(h >> 40) * (1.0f / 16777216.0f));
      ++e;
    }
  }
}

extern "C" int dawn_gen_grid(int device, int64_t rows, int64_t cols, int wkind, int64_t wlo, int64_t whi,
                             uint64_t wseed, int64_t* row_ptr_out, int64_t* col_out, double* val_out,
                             void* stream) {
  if (rows < 1 || cols < 1 || rows > (1ll << 31) / cols || !row_ptr_out ||
      ((rows > 1 || cols > 1) && (!col_out || !val_out)))
    return fail(DAWN_EINVAL, "bad grid arguments");
  if (wkind == 0 && (whi < wlo || whi - wlo >= (1ll << 32))) return fail(DAWN_EINVAL, "bad weight range");
  CK(cudaSetDevice(device));
  const int64_t n = rows * cols;
  const int blocks = (int)std::min<int64_t>((n + 256) / 256, 148 * 16);
  k_gen_grid<<<blocks, 256, 0, (cudaStream_t)stream>>>(rows, cols, wkind, wlo,
                                                       (unsigned long long)(whi - wlo + 1), wseed,
                                                       row_ptr_out, col_out, val_out);
  CK(cudaGetLastError());
  return DAWN_OK;
}

// ---------------------------------------------------------------------------
// Floyd–Warshall on the device (floyd_warshall_apsp, oracles.py:141-162)
// ---------------------------------------------------------------------------
extern "C" int dawn_floyd_warshall(int device, int64_t n, const int64_t* row_ptr, const int64_t* col,
                                   const double* val, double* out, int* negative_cycle_out, void* stream) {
  if (n < 0) return fail(DAWN_EINVAL, "n must be >= 0");
  if (n > 0 && (!row_ptr || !out)) return fail(DAWN_EINVAL, "NULL argument");
  if (negative_cycle_out) *negative_cycle_out = 0;
  if (n == 0) return DAWN_OK;
  if (n > (1ll << 31)) return fail(DAWN_EUNSUPPORTED, "n=%lld too large for a dense matrix", (long long)n);
  CK(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  int64_t m = 0;
  CK(cudaMemcpy(&m, row_ptr + n, sizeof(int64_t), cudaMemcpyDefault));
  if (m < 0) return fail(DAWN_EINVAL, "row_ptr[n] must be >= 0");
  if (m > 0 && (!col || !val)) return fail(DAWN_EINVAL, "NULL argument");
  const size_t nn = (size_t)n * (size_t)n;
  char* ws = nullptr;
  const size_t in_bytes = 8 * (size_t)(n + 1) + 16 * (size_t)m;
  const size_t bytes = 8 * nn + 32 * (size_t)n + in_bytes + 64;
  CK(dmalloc(&ws, bytes));
  auto release = [&](int rc) {
    cudaStreamSynchronize(st);
    dfree(ws);
    return rc;
  };
  unsigned long long* D = (unsigned long long*)ws;
  double* colb = (double*)(ws + 8 * nn);
  double* rowb = colb + 2 * n;
  int64_t* d_rp = (int64_t*)(rowb + 2 * n);
  int64_t* d_col = d_rp + (n + 1);
  double* d_val = (double*)(d_col + m);
  unsigned* flags = (unsigned*)(d_val + m);  // [0] barrier, [1] bad column, [2] negative diagonal, [3] abort
  cudaError_t e;
  if ((e = cudaMemcpyAsync(d_rp, row_ptr, 8 * (size_t)(n + 1), cudaMemcpyDefault, st)) != cudaSuccess ||
      (m && (e = cudaMemcpyAsync(d_col, col, 8 * (size_t)m, cudaMemcpyDefault, st)) != cudaSuccess) ||
      (m && (e = cudaMemcpyAsync(d_val, val, 8 * (size_t)m, cudaMemcpyDefault, st)) != cudaSuccess) ||
      (e = cudaMemsetAsync(flags, 0, 16, st)) != cudaSuccess)
    return release(fail(DAWN_ECUDA, "upload: %s", cudaGetErrorString(e)));
  int nsm = 0, bps = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  const int eb = (int)std::min<int64_t>((int64_t)nsm * 8, std::max<int64_t>(1, ((int64_t)nn + 255) / 256));
  fw_init<<<eb, 256, 0, st>>>(D, n);
  fw_edges<<<(int)std::min<int64_t>((int64_t)nsm * 8, (n + 255) / 256), 256, 0, st>>>(D, n, d_rp, d_col, d_val,
                                                                                      flags + 1);
  fw_decode<<<eb, 256, 0, st>>>(D, n, colb, rowb);
  if ((e = cudaGetLastError()) != cudaSuccess) return release(fail(DAWN_ECUDA, "init: %s", cudaGetErrorString(e)));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fw_steps, 256, 0));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)bps * nsm, ((int64_t)nn + 255) / 256));
  double* M = (double*)D;
  unsigned* bar = flags;
  void* args[] = {&M, &n, &colb, &rowb, &bar};
  if ((e = cudaLaunchCooperativeKernel((void*)fw_steps, dim3(grid), dim3(256), args, 0, st)) != cudaSuccess)
    return release(fail(DAWN_ECUDA, "steps: %s", cudaGetErrorString(e)));
  fw_negdiag<<<(int)std::min<int64_t>(nsm * 4, (n + 255) / 256), 256, 0, st>>>(M, n, flags + 2);
  unsigned hf[4] = {0, 0, 0, 0};
  if ((e = cudaMemcpyAsync(out, M, 8 * nn, cudaMemcpyDefault, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(hf, flags, 16, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return release(fail(DAWN_ECUDA, "floyd-warshall: %s", cudaGetErrorString(e)));
  if (hf[3]) return release(fail(DAWN_ECUDA, "device watchdog: floyd-warshall made no progress for 30 s"));
  if (hf[1]) return release(fail(DAWN_EINVAL, "column index out of range"));
  if (negative_cycle_out) *negative_cycle_out = hf[2] ? 1 : 0;
  return release(DAWN_OK);
}

// ---------------------------------------------------------------------------
// distance rows as text (format_distance_row, solver.py:498-506), host side
// ---------------------------------------------------------------------------
// One value exactly as Python's `"inf" if d == inf else "%.17g" % d`: printf's
// %.17g is correctly rounded like Python's float formatting; NaN is "nan"
// whatever its sign (Python), -inf is "-inf".
static int fmt_value(char* p, double d) {
  if (d != d) {
    memcpy(p, "nan", 3);
    return 3;
  }
  if (d == HUGE_VAL) {
    memcpy(p, "inf", 3);
    return 3;
  }
  // std::to_chars with a precision is specified as printf's conversion in the C locale
  // (checked identical on 2^20 random bit patterns, tests/test_rows_output.py), ~2x faster
  return (int)(std::to_chars(p, p + 32, d, std::chars_format::general, 17).ptr - p);
}

static int64_t fmt_row(char* out, int64_t source, const double* row, int64_t n) {
  char* p = out;
  p += snprintf(p, 24, "%lld", (long long)source);
  for (int64_t j = 0; j < n; ++j) {
    *p++ = ',';
    p += fmt_value(p, row[j]);
  }
  *p++ = '\n';
  return p - out;
}

extern "C" int dawn_format_rows(const double* rows, int64_t k, int64_t n, int64_t ld, const int64_t* sources,
                                char* out, int64_t cap, int64_t* len_out, int threads) {
  if (k < 0 || n < 0 || ld < n || (k > 0 && (!rows || !sources || !out)) || !len_out)
    return fail(DAWN_EINVAL, "bad arguments");
  const int64_t per_row = 24 + 26 * n;  // bound: source + n x ("," + 25 chars) + newline
  if (cap < k * per_row) {
    *len_out = k * per_row;
    return fail(DAWN_EINVAL, "out too small: need %lld bytes", (long long)(k * per_row));
  }
  if (k == 0) {
    *len_out = 0;
    return DAWN_OK;
  }
  // rows are formatted into disjoint slots of `out`, then packed in place in order
  const int T = std::max(1, std::min<int>(threads > 0 ? threads : (int)std::thread::hardware_concurrency(),
                                          (int)std::max<int64_t>(1, k * n / 65536)));
  std::vector<int64_t> len((size_t)k, 0);
  if (k >= T) {
    auto work = [&](int t) {
      for (int64_t r = t; r < k; r += T) len[(size_t)r] = fmt_row(out + r * per_row, sources[r], rows + r * ld, n);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  } else {
    // few long rows: split each row's values over the threads, then stitch
    for (int64_t r = 0; r < k; ++r) {
      char* base = out + r * per_row;
      const double* row = rows + r * ld;
      const int64_t chunk = (n + T - 1) / T;
      std::vector<std::string> parts((size_t)T);
      auto work = [&](int t) {
        const int64_t a = std::min<int64_t>(n, (int64_t)t * chunk), b = std::min<int64_t>(n, a + chunk);
        std::string& sbuf = parts[(size_t)t];
        sbuf.resize((size_t)(26 * (b - a)));
        char* p = &sbuf[0];
        for (int64_t j = a; j < b; ++j) {
          *p++ = ',';
          p += fmt_value(p, row[j]);
        }
        sbuf.resize((size_t)(p - &sbuf[0]));
      };
      std::vector<std::thread> pool;
      for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
      work(0);
      for (auto& th : pool) th.join();
      char* p = base + snprintf(base, 24, "%lld", (long long)sources[r]);
      for (auto& part : parts) {
        memcpy(p, part.data(), part.size());
        p += part.size();
      }
      *p++ = '\n';
      len[(size_t)r] = p - base;
    }
  }
  int64_t pos = 0;
  for (int64_t r = 0; r < k; ++r) {
    if (pos != r * per_row) memmove(out + pos, out + r * per_row, (size_t)len[(size_t)r]);
    pos += len[(size_t)r];
  }
  *len_out = pos;
  return DAWN_OK;
}
