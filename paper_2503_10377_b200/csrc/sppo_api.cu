// C-ABI runtime of the SPPO hot path (include/sppo.h): argument validation,
// FIRST/LAST window-coverage tracking, TMA descriptor cache, dispatch to the
// kernels, pinned host arena and the D2H/H2D copy streams of the two-level
// activation manager, host plan helpers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/sppo.h"
#include "internal.h"

using namespace sppo;

// ---------------------------------------------------------------- errors
namespace {
thread_local char g_err[512] = "";

sppo_status fail(sppo_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

sppo_status cuda_fail(cudaError_t e, const char* what) {
  return fail(SPPO_E_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define SPPO_CUDA(call, what)                      \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

// ---------------------------------------------------------------- TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct DescKey {
  const void* ptr;
  int64_t rows;
  int32_t heads, d, box_rows, elem;
  bool operator==(const DescKey& o) const {
    return ptr == o.ptr && rows == o.rows && heads == o.heads && d == o.d && box_rows == o.box_rows &&
           elem == o.elem;
  }
};
struct DescKeyHash {
  size_t operator()(const DescKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<int64_t>()(k.rows * 1000003 + k.heads * 131 + k.d * 7 + k.box_rows * 3 + k.elem) +
         0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
  }
};

// TMA descriptors live in ONE persistent device table of kDescSlots maps.  A
// map (key: pointer + shape) is encoded on the host and uploaded once, the
// first time a call needs it: one cudaMemcpyAsync of the call's new maps on
// the launch stream, followed by an event.  Later calls that hit the slot from
// another stream make their stream wait on that event until its completion has
// been observed once, so a kernel never reads a table entry whose upload is
// unordered with it.  In the steady state (same buffers every step)
// no call uploads anything, so no descriptor copy ever queues behind the large
// offload / prefetch copies on the copy engines.  When a call's new maps do not
// fit, the table is recycled BEFORE any slot of that call is resolved, after
// every stream that launched from the table has drained (host wait; rare).
constexpr int kSchedSlots = 1024;          // persistent-bwd item counters (one per launch in flight)
constexpr int kDescSlots = 16384;          // kernels take uint16_t slot indices
constexpr int kDescCallMax = 8 + 4 * kMaxWindow;  // multi-chunk forward: K, V, Q, O of up to kMaxWindow chunks
constexpr int kUploadEvents = 64;

struct Coverage {
  int32_t chunk;
  std::vector<uint8_t> seen;  // 0..chunk
};

}  // namespace

struct sppo_ctx_s {
  int device = 0;
  cudaStream_t d2h = nullptr, h2d = nullptr;
  cudaEvent_t ev_prod = nullptr, ev_cons = nullptr, ev_copy = nullptr;
  // TMA descriptors: persistent device table + pinned host mirror, key -> slot,
  // per-slot upload record (event id, its generation, upload stream, observed done)
  CUtensorMap* desc_dev = nullptr;
  // persistent bwd item counters: one int per launch, taken round-robin and zeroed on
  // the launch stream just before the kernel (kSchedSlots launches may be in flight)
  int* sched = nullptr;
  unsigned sched_next = 0;
  CUtensorMap* desc_host = nullptr;
  std::unordered_map<DescKey, int, DescKeyHash> desc_slot;
  struct SlotUpload {
    int ev = -1;
    uint32_t gen = 0;
    cudaStream_t stream = nullptr;
    bool done = true;
  };
  std::vector<SlotUpload> slot_up;
  int desc_next = 0;
  cudaEvent_t up_ev[kUploadEvents] = {};
  uint32_t up_gen[kUploadEvents] = {};
  bool up_live[kUploadEvents] = {};
  int up_next = 0;
  std::vector<cudaStream_t> desc_streams;  // streams that launched from the table since the last recycle
  // window coverage per (direction, q pointer)
  std::unordered_map<const void*, Coverage> cov_fwd, cov_bwd;
  // host arena: ptr -> bytes (mmap + mbind + cudaHostRegister) or 0 (cudaHostAlloc fallback)
  std::unordered_map<void*, size_t> host_allocs;
  int numa_node = -1;  // NUMA node of the GPU (sysfs), -1 unknown
  std::mutex mu;
  // debug tracing (env SPPO_TRACE=<file>, SPPO_TRACE_CHUNK=<i>, SPPO_TRACE_KIND=fwd|bwd):
  // clock64 stamps of CTA (0,0) of one launch, dumped by sppo_ctx_sync
  unsigned long long* trace = nullptr;
  int trace_chunk = -1;
  int trace_bwd = 1;
  int trace_life = 0;  // SPPO_TRACE_LIFE: per-CTA lifetime stamps of the traced bwd launch
};

namespace {
constexpr size_t kTraceWords = (size_t)sppo::kTraceIters * sppo::kTraceSlots;

unsigned long long* trace_for(sppo_ctx ctx, int chunk, bool bwd) {
  if (!ctx->trace) return nullptr;
  return (chunk == ctx->trace_chunk && (int)bwd == ctx->trace_bwd) ? ctx->trace : nullptr;
}

void trace_dump(sppo_ctx ctx) {
  const char* path = getenv("SPPO_TRACE");
  if (!ctx->trace || !path) return;
  if (ctx->trace_life) {
    std::vector<unsigned long long> h(sppo::kLifeWords);
    if (cudaMemcpy(h.data(), ctx->trace, sppo::kLifeWords * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
    FILE* f = fopen(path, "w");
    if (!f) return;
    for (size_t c = 0; c < sppo::kLifeWords / sppo::kLifeSlots; ++c) {
      const unsigned long long* r = &h[c * sppo::kLifeSlots];
      if (r[0] == 0) continue;
      fprintf(f, "%zu", c);
      for (int s = 0; s < sppo::kLifeSlots; ++s) fprintf(f, " %llu", r[s]);
      fprintf(f, "\n");
    }
    fclose(f);
    return;
  }
  std::vector<unsigned long long> h(kTraceWords);
  if (cudaMemcpy(h.data(), ctx->trace, kTraceWords * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  FILE* f = fopen(path, "w");
  if (!f) return;
  for (int it = 0; it < sppo::kTraceIters; ++it) {
    bool any = false;
    for (int s = 0; s < sppo::kTraceSlots; ++s) any |= h[it * sppo::kTraceSlots + s] != 0;
    if (!any) continue;
    fprintf(f, "%d", it);
    for (int s = 0; s < sppo::kTraceSlots; ++s) fprintf(f, " %llu", h[it * sppo::kTraceSlots + s]);
    fprintf(f, "\n");
  }
  fclose(f);
}
}  // namespace

namespace {

// Encoded tensor map of a token-major [rows, heads, d] tensor of bf16 (elem = 2)
// or fp32 (elem = 4), tiled as boxes of {128 B of d (SWIZZLE_128B), 1 head,
// box_rows}.
sppo_status encode_desc(const DescKey& key, CUtensorMap* out) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(SPPO_E_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  const int elem = key.elem, d = key.d;
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)key.heads, (cuuint64_t)key.rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * elem, (cuuint64_t)key.heads * d * elem};
  cuuint32_t box[3] = {(cuuint32_t)(128 / elem), 1, (cuuint32_t)key.box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(key.ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPPO_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SPPO_OK;
}

// Waits until every launch that may read the descriptor table has finished:
// an event recorded on each stream that launched from it since the last
// recycle (host wait), or the whole device if a stream cannot be recorded.
sppo_status drain_desc_streams(sppo_ctx ctx) {
  cudaEvent_t ev;
  SPPO_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "descriptor recycle");
  bool ok = true;
  for (cudaStream_t st : ctx->desc_streams)
    ok = ok && cudaEventRecord(ev, st) == cudaSuccess && cudaEventSynchronize(ev) == cudaSuccess;
  cudaEventDestroy(ev);
  if (!ok) {
    cudaGetLastError();
    SPPO_CUDA(cudaDeviceSynchronize(), "descriptor recycle");
  }
  for (int e = 0; e < kUploadEvents; ++e) ctx->up_live[e] = false;
  ctx->desc_streams.clear();
  return SPPO_OK;
}

// The descriptor set of one launch.  Usage: add() every map the kernel reads
// (returns a request index), resolve(stream) once (uploads new maps, orders the
// stream after pending uploads), then slot(index).  A failure leaves nothing
// enqueued except, possibly, an upload of maps into free slots.
struct DescBlock {
  sppo_ctx ctx = nullptr;
  std::vector<DescKey> keys;
  std::vector<int> slots;
  void open(sppo_ctx c) {
    ctx = c;
    keys.clear();
    slots.clear();
  }
  int add(const void* ptr, int64_t rows, int heads, int d, int box_rows, int elem = 2) {
    keys.push_back(DescKey{ptr, rows, heads, d, box_rows, elem});
    return (int)keys.size() - 1;
  }
  int slot(int i) const { return slots[i]; }
  const void* table() const { return ctx->desc_dev; }
  sppo_status resolve(cudaStream_t stream) {
    if ((int)keys.size() > kDescCallMax) return fail(SPPO_E_UNSUPPORTED, "too many descriptors in one launch");
    // pass 1: how many new maps (deduplicated); recycle first if they do not fit
    std::vector<DescKey> fresh;
    for (const DescKey& k : keys)
      if (!ctx->desc_slot.count(k) && std::find(fresh.begin(), fresh.end(), k) == fresh.end()) fresh.push_back(k);
    if (ctx->desc_next + (int)fresh.size() > kDescSlots) {
      sppo_status s = drain_desc_streams(ctx);
      if (s) return s;
      ctx->desc_slot.clear();
      ctx->desc_next = 0;
    }
    // pass 2: encode the new maps into consecutive slots of the host mirror
    const int first = ctx->desc_next;
    for (size_t f = 0; f < fresh.size(); ++f) {
      sppo_status s = encode_desc(fresh[f], &ctx->desc_host[first + f]);
      if (s) return s;
    }
    if (!fresh.empty()) {
      // one upload of the new run, then its event (an event is re-recorded only after
      // its previous upload is known complete, so a slot's generation check is exact)
      const int e = ctx->up_next;
      ctx->up_next = (e + 1) % kUploadEvents;
      if (ctx->up_live[e]) SPPO_CUDA(cudaEventSynchronize(ctx->up_ev[e]), "descriptor upload event reuse");
      SPPO_CUDA(cudaMemcpyAsync(ctx->desc_dev + first, ctx->desc_host + first, sizeof(CUtensorMap) * fresh.size(),
                                cudaMemcpyHostToDevice, stream),
                "descriptor upload");
      SPPO_CUDA(cudaEventRecord(ctx->up_ev[e], stream), "descriptor upload event");
      ++ctx->up_gen[e];
      ctx->up_live[e] = true;
      for (size_t f = 0; f < fresh.size(); ++f) {
        const int sl = first + (int)f;
        ctx->desc_slot[fresh[f]] = sl;
        ctx->slot_up[sl] = sppo_ctx_s::SlotUpload{e, ctx->up_gen[e], stream, false};
      }
      ctx->desc_next = first + (int)fresh.size();
    }
    // pass 3: slots; order this stream after uploads issued on other streams
    slots.resize(keys.size());
    std::vector<int> waited;
    for (size_t i = 0; i < keys.size(); ++i) {
      const int sl = ctx->desc_slot[keys[i]];
      slots[i] = sl;
      sppo_ctx_s::SlotUpload& u = ctx->slot_up[sl];
      if (u.done || u.stream == stream) continue;
      if (u.gen != ctx->up_gen[u.ev] || cudaEventQuery(ctx->up_ev[u.ev]) == cudaSuccess) {
        u.done = true;  // the event was re-recorded after a completed wait, or has completed
        continue;
      }
      cudaGetLastError();  // cudaErrorNotReady from the query is not an error
      if (std::find(waited.begin(), waited.end(), u.ev) == waited.end()) {
        SPPO_CUDA(cudaStreamWaitEvent(stream, ctx->up_ev[u.ev], 0), "descriptor upload ordering");
        waited.push_back(u.ev);
      }
    }
    if (std::find(ctx->desc_streams.begin(), ctx->desc_streams.end(), stream) == ctx->desc_streams.end())
      ctx->desc_streams.push_back(stream);
    return SPPO_OK;
  }
};

// ---------------------------------------------------------------- validation
sppo_status check_layout(const sppo_layout* L, int32_t chunk) {
  if (!L) return fail(SPPO_E_ARG, "layout is NULL");
  if (!L->offsets) return fail(SPPO_E_ARG, "layout.offsets is NULL");
  if (L->heads < 1) return fail(SPPO_E_SHAPE, "layout.heads = %d < 1", L->heads);
  if (L->dtype != SPPO_BF16 && L->dtype != SPPO_FP32) return fail(SPPO_E_ARG, "layout.dtype = %d", L->dtype);
  if (L->dtype == SPPO_FP32 && L->head_dim != 32 && L->head_dim != 64 && L->head_dim != 128)
    return fail(SPPO_E_UNSUPPORTED, "fp32 path supports head_dim 32/64/128, got %d", L->head_dim);
  if (L->dtype == SPPO_BF16 && L->head_dim != 128)
    return fail(SPPO_E_UNSUPPORTED, "bf16 tensor-core path supports head_dim 128, got %d", L->head_dim);
  if (L->num_chunks < 1) return fail(SPPO_E_SHAPE, "layout.num_chunks = %d < 1", L->num_chunks);
  if (L->offsets[0] != 0) return fail(SPPO_E_SHAPE, "offsets[0] = %lld != 0", (long long)L->offsets[0]);
  for (int i = 0; i < L->num_chunks; ++i)
    if (L->offsets[i + 1] <= L->offsets[i])
      return fail(SPPO_E_SHAPE, "offsets not strictly increasing at %d", i);
  if (L->offsets[L->num_chunks] > (int64_t)INT32_MAX) return fail(SPPO_E_SHAPE, "S exceeds 2^31-1");
  if (!(L->scale >= 0.f) || !isfinite(L->scale)) return fail(SPPO_E_ARG, "scale must be finite and >= 0");
  if (chunk < 0 || chunk >= L->num_chunks)
    return fail(SPPO_E_SHAPE, "chunk %d outside [0, %d)", chunk, L->num_chunks);
  return SPPO_OK;
}

sppo_status check_kv(const sppo_layout* L, int32_t chunk, const sppo_kv_set* kv, const Coverage* cov,
                     bool first, bool last) {
  if (!kv) return fail(SPPO_E_ARG, "kv set is NULL");
  if (kv->n < 1) return fail(SPPO_E_ARG, "kv.n = %d < 1", kv->n);
  if (kv->n > kMaxWindow) return fail(SPPO_E_UNSUPPORTED, "kv.n = %d > %d: split the window", kv->n, kMaxWindow);
  if (!kv->ids || !kv->k || !kv->v) return fail(SPPO_E_ARG, "kv arrays are NULL");
  std::vector<uint8_t> seen(chunk + 1, 0);
  if (!first && cov) seen = cov->seen;
  for (int c = 0; c < kv->n; ++c) {
    const int j = kv->ids[c];
    if (j < 0 || j > chunk) return fail(SPPO_E_SHAPE, "kv id %d not in [0, %d]", j, chunk);
    if (!kv->k[c] || !kv->v[c]) return fail(SPPO_E_ARG, "kv buffer %d is NULL", c);
    if (!aligned16(kv->k[c]) || !aligned16(kv->v[c])) return fail(SPPO_E_ALIGN, "kv buffer %d not 16B aligned", c);
    if (seen[j]) return fail(SPPO_E_STATE, "chunk %d appears twice in the windows of chunk %d", j, chunk);
    seen[j] = 1;
  }
  if (last)
    for (int j = 0; j <= chunk; ++j)
      if (!seen[j]) return fail(SPPO_E_STATE, "LAST window of chunk %d leaves chunk %d uncovered", chunk, j);
  (void)L;
  return SPPO_OK;
}

// Applies the window to the coverage map (called only after a successful enqueue).
void commit_coverage(std::unordered_map<const void*, Coverage>& m, const void* key, int32_t chunk,
                     const sppo_kv_set* kv, bool first, bool last) {
  if (last) {
    m.erase(key);
    return;
  }
  Coverage& c = m[key];
  if (first) {
    c.chunk = chunk;
    c.seen.assign(chunk + 1, 0);
  }
  for (int i = 0; i < kv->n; ++i) c.seen[kv->ids[i]] = 1;
}

sppo_status lookup_coverage(std::unordered_map<const void*, Coverage>& m, const void* key, int32_t chunk,
                            bool first, const Coverage** out) {
  *out = nullptr;
  auto it = m.find(key);
  if (first) {
    if (it != m.end()) m.erase(it);  // a new FIRST abandons an unfinished chunk state
    return SPPO_OK;
  }
  if (it == m.end() || it->second.chunk != chunk)
    return fail(SPPO_E_STATE, "window of chunk %d without FIRST (no open state for this q)", chunk);
  *out = &it->second;
  return SPPO_OK;
}

void fill_window(const sppo_layout* L, const sppo_kv_set* kv, KvWindow* w) {
  w->n = kv->n;
  for (int c = 0; c < kv->n; ++c) {
    const int j = kv->ids[c];
    w->start[c] = (int32_t)L->offsets[j];
    w->len[c] = (int32_t)(L->offsets[j + 1] - L->offsets[j]);
    w->k[c] = kv->k[c];
    w->v[c] = kv->v[c];
  }
}

}  // namespace

namespace {
// NUMA node of a GPU from sysfs (/sys/bus/pci/devices/<bus id>/numa_node), -1 if unknown.
int gpu_numa_node(int device) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
  unsigned dom = 0, b = 0, d = 0, f = 0;
  if (sscanf(bus, "%x:%x:%x.%x", &dom, &b, &d, &f) != 4) return -1;
  char path[128];
  snprintf(path, sizeof path, "/sys/bus/pci/devices/%04x:%02x:%02x.%x/numa_node", dom & 0xffffu, b, d, f);
  FILE* fp = fopen(path, "r");
  if (!fp) return -1;
  int node = -1;
  if (fscanf(fp, "%d", &node) != 1) node = -1;
  fclose(fp);
  return node;
}

// Page-locked host memory placed on `node` (P:472 [§7]: "bind the NUMA node ...
// page-locked memory"): anonymous mapping, mbind(MPOL_PREFERRED) before first
// touch, then cudaHostRegister (which faults the pages in, on that node).
void* numa_pinned_alloc(size_t bytes, int node) {
  if (node < 0 || node >= 64) return nullptr;
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return nullptr;
  unsigned long mask = 1ul << node;
  const int kMpolPreferred = 1;
  if (syscall(SYS_mbind, p, bytes, kMpolPreferred, &mask, (unsigned long)(8 * sizeof mask), 0u) != 0) {
    munmap(p, bytes);
    return nullptr;
  }
  if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) != cudaSuccess) {
    cudaGetLastError();
    munmap(p, bytes);
    return nullptr;
  }
  return p;
}
}  // namespace

int sppo::api_fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return status;
}

// ================================================================ C ABI
extern "C" {

int32_t sppo_version(void) { return 100; }

const char* sppo_last_error(void) { return g_err; }

sppo_status sppo_ctx_create(int device, sppo_ctx* out) {
  if (!out) return fail(SPPO_E_ARG, "out is NULL");
  *out = nullptr;
  int n = 0;
  SPPO_CUDA(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(SPPO_E_ARG, "device %d not in [0, %d)", device, n);
  SPPO_CUDA(cudaSetDevice(device), "cudaSetDevice");
  sppo_ctx c = new sppo_ctx_s();
  c->device = device;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->ev_prod, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->ev_cons, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaMalloc(&c->desc_dev, sizeof(CUtensorMap) * kDescSlots)) != cudaSuccess ||
      (e = cudaMalloc(&c->sched, sizeof(int) * kSchedSlots)) != cudaSuccess ||
      (e = cudaHostAlloc(&c->desc_host, sizeof(CUtensorMap) * kDescSlots, cudaHostAllocDefault)) !=
          cudaSuccess) {
    sppo_ctx_destroy(c);
    return cuda_fail(e, "sppo_ctx_create");
  }
  c->slot_up.resize(kDescSlots);
  for (int b = 0; b < kUploadEvents; ++b)
    if ((e = cudaEventCreateWithFlags(&c->up_ev[b], cudaEventDisableTiming)) != cudaSuccess) {
    sppo_ctx_destroy(c);
    return cuda_fail(e, "sppo_ctx_create");
  }
  c->numa_node = gpu_numa_node(device);
  if (getenv("SPPO_TRACE")) {
    const char* ch = getenv("SPPO_TRACE_CHUNK");
    const char* kind = getenv("SPPO_TRACE_KIND");
    c->trace_chunk = ch ? atoi(ch) : 0;
    c->trace_bwd = (kind && strcmp(kind, "fwd") == 0) ? 0 : 1;
    c->trace_life = getenv("SPPO_TRACE_LIFE") && c->trace_bwd ? 1 : 0;
    const size_t words = c->trace_life ? sppo::kLifeWords : kTraceWords;
    if (cudaMalloc(&c->trace, words * 8) != cudaSuccess || cudaMemset(c->trace, 0, words * 8) != cudaSuccess)
      c->trace = nullptr;
  }
  *out = c;
  return SPPO_OK;
}

sppo_status sppo_ctx_destroy(sppo_ctx c) {
  if (!c) return fail(SPPO_E_ARG, "ctx is NULL");
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->host_allocs) {
    if (kv.second) {
      cudaHostUnregister(kv.first);
      munmap(kv.first, kv.second);
    } else {
      cudaFreeHost(kv.first);
    }
  }
  if (c->d2h) cudaStreamDestroy(c->d2h);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->ev_prod) cudaEventDestroy(c->ev_prod);
  if (c->ev_cons) cudaEventDestroy(c->ev_cons);
  if (c->ev_copy) cudaEventDestroy(c->ev_copy);
  for (int b = 0; b < kUploadEvents; ++b)
    if (c->up_ev[b]) cudaEventDestroy(c->up_ev[b]);
  if (c->desc_dev) cudaFree(c->desc_dev);
  if (c->sched) cudaFree(c->sched);
  if (c->desc_host) cudaFreeHost(c->desc_host);
  if (c->trace) cudaFree(c->trace);
  delete c;
  return SPPO_OK;
}

sppo_status sppo_ctx_sync(sppo_ctx c) {
  if (!c) return fail(SPPO_E_ARG, "ctx is NULL");
  SPPO_CUDA(cudaSetDevice(c->device), "cudaSetDevice");
  SPPO_CUDA(cudaDeviceSynchronize(), "device fault");
  SPPO_CUDA(cudaGetLastError(), "device fault");
  trace_dump(c);
  return SPPO_OK;
}

// ---------------------------------------------------------------- forward
sppo_status sppo_attn_fwd(sppo_ctx ctx, const sppo_layout* L, int32_t chunk, const void* q, const sppo_kv_set* kv,
                          int32_t flags, const sppo_fwd_state* st, void* o, float* lse, void* stream) {
  if (!ctx) return fail(SPPO_E_ARG, "ctx is NULL");
  sppo_status s = check_layout(L, chunk);
  if (s) return s;
  if (flags & ~(SPPO_FIRST | SPPO_LAST)) return fail(SPPO_E_ARG, "unknown flags 0x%x", flags);
  const bool first = flags & SPPO_FIRST, last = flags & SPPO_LAST;
  if (!q) return fail(SPPO_E_ARG, "q is NULL");
  if (!aligned16(q)) return fail(SPPO_E_ALIGN, "q not 16B aligned");
  if (last && (!o || !lse)) return fail(SPPO_E_ARG, "o/lse NULL on LAST");
  if (last && (!aligned16(o) || !aligned4(lse))) return fail(SPPO_E_ALIGN, "o not 16B / lse not 4B aligned");
  const bool need_state = !(first && last);
  if (need_state && (!st || !st->o_acc || !st->m || !st->l))
    return fail(SPPO_E_ARG, "split windows need a carry state (o_acc, m, l)");
  if (need_state && (!aligned16(st->o_acc) || !aligned4(st->m) || !aligned4(st->l)))
    return fail(SPPO_E_ALIGN, "carry state: o_acc needs 16B, m/l 4B alignment");
  std::lock_guard<std::mutex> lock(ctx->mu);
  const Coverage* cov = nullptr;
  if ((s = lookup_coverage(ctx->cov_fwd, q, chunk, first, &cov))) return s;
  if ((s = check_kv(L, chunk, kv, cov, first, last))) return s;
  SPPO_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");

  cudaStream_t strm = (cudaStream_t)stream;
  FwdParams p{};
  p.heads = L->heads;
  p.d = L->head_dim;
  p.q_start = (int32_t)L->offsets[chunk];
  p.q_len = (int32_t)(L->offsets[chunk + 1] - L->offsets[chunk]);
  p.scale = L->scale > 0.f ? L->scale : 1.f / sqrtf((float)L->head_dim);
  p.first = first;
  p.last = last;
  p.q = q;
  p.o = o;
  p.lse = lse;
  p.trace = trace_for(ctx, chunk, false);
  if (st) {
    p.o_acc = st->o_acc;
    p.m = st->m;
    p.l = st->l;
  }
  cudaError_t e;
  if (L->dtype == SPPO_FP32) {
    KvWindow w;  // per call: no state shared between contexts or threads
    fill_window(L, kv, &w);
    e = launch_fwd_simt_f32(p, w, strm);
  } else {
    Sm100Fwd a{};
    a.p = p;
    a.n = kv->n;
    DescBlock db;
    db.open(ctx);
    const int rq = db.add(q, p.q_len, p.heads, p.d, 128);
    const int ro = last ? db.add(o, p.q_len, p.heads, p.d, 128) : -1;
    std::vector<int> rk(kv->n), rv(kv->n);
    // kernel contract: the diagonal chunk (id == chunk), if present, is visited last
    std::vector<int> order;
    for (int c = 0; c < kv->n; ++c)
      if (kv->ids[c] != chunk) order.push_back(c);
    for (int c = 0; c < kv->n; ++c)
      if (kv->ids[c] == chunk) order.push_back(c);
    for (int oc = 0; oc < kv->n; ++oc) {
      const int c = order[oc];
      const int j = kv->ids[c];
      const int64_t len = L->offsets[j + 1] - L->offsets[j];
      a.start[oc] = (int32_t)L->offsets[j];
      a.len[oc] = (int32_t)len;
      rk[oc] = db.add(kv->k[c], len, p.heads, p.d, 128);
      rv[oc] = db.add(kv->v[c], len, p.heads, p.d, 128);
    }
    if ((s = db.resolve(strm))) return s;
    a.q_slot = db.slot(rq);
    a.o_slot = last ? db.slot(ro) : -1;
    for (int oc = 0; oc < kv->n; ++oc) {
      a.slots.k[oc] = (uint16_t)db.slot(rk[oc]);
      a.slots.v[oc] = (uint16_t)db.slot(rv[oc]);
    }
    a.desc_table = db.table();
    e = launch_fwd_sm100(a, strm);
  }
  if (e == cudaErrorNotSupported) return fail(SPPO_E_UNSUPPORTED, "this request is not implemented by the sm_100a kernels");
  if (e != cudaSuccess) return cuda_fail(e, "sppo_attn_fwd launch");
  commit_coverage(ctx->cov_fwd, q, chunk, kv, first, last);
  return SPPO_OK;
}

// ---------------------------------------------------------------- forward of several chunks
sppo_status sppo_attn_fwd_chunks(sppo_ctx ctx, const sppo_layout* L, int32_t i0, int32_t i1, const void* const* q,
                                 const sppo_kv_set* kv, void* const* o, float* const* lse, void* stream) {
  if (!ctx) return fail(SPPO_E_ARG, "ctx is NULL");
  sppo_status s = check_layout(L, i0);
  if (s) return s;
  if (i1 <= i0 || i1 > L->num_chunks) return fail(SPPO_E_SHAPE, "chunk range [%d, %d) invalid", i0, i1);
  if (i1 - i0 > kMaxWindow) return fail(SPPO_E_UNSUPPORTED, "more than %d chunks in one launch", kMaxWindow);
  if (L->dtype != SPPO_BF16) return fail(SPPO_E_UNSUPPORTED, "multi-chunk forward: bf16 only");
  if (!q || !o || !lse) return fail(SPPO_E_ARG, "q/o/lse arrays are NULL");
  if (!kv || !kv->ids || !kv->k || !kv->v) return fail(SPPO_E_ARG, "kv set is NULL");
  if (kv->n != i1) return fail(SPPO_E_ARG, "kv must hold exactly chunks 0..%d", i1 - 1);
  for (int c = 0; c < kv->n; ++c) {
    if (kv->ids[c] != c) return fail(SPPO_E_ARG, "kv ids must be 0..%d in ascending order", i1 - 1);
    if (!kv->k[c] || !kv->v[c]) return fail(SPPO_E_ARG, "kv buffer %d is NULL", c);
    if (!aligned16(kv->k[c]) || !aligned16(kv->v[c])) return fail(SPPO_E_ALIGN, "kv buffer %d not 16B aligned", c);
  }
  for (int k = 0; k < i1 - i0; ++k) {
    if (!q[k] || !o[k] || !lse[k]) return fail(SPPO_E_ARG, "q/o/lse %d is NULL", k);
    if (!aligned16(q[k]) || !aligned16(o[k]) || !aligned4(lse[k])) return fail(SPPO_E_ALIGN, "q/o/lse %d misaligned", k);
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  SPPO_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t strm = (cudaStream_t)stream;
  Sm100Fwd a{};
  FwdParams& p = a.p;
  p.heads = L->heads;
  p.d = L->head_dim;
  p.scale = L->scale > 0.f ? L->scale : 1.f / sqrtf((float)L->head_dim);
  p.first = 1;
  p.last = 1;
  p.q_start = (int32_t)L->offsets[i0];
  p.q_len = (int32_t)(L->offsets[i0 + 1] - L->offsets[i0]);
  p.trace = trace_for(ctx, i1 - 1, false);
  a.n = kv->n;
  a.nq = i1 - i0;
  a.q0 = i0;
  DescBlock db;
  db.open(ctx);
  std::vector<int> rk(kv->n), rv(kv->n), rq(a.nq), ro(a.nq);
  for (int c = 0; c < kv->n; ++c) {
    const int64_t len = L->offsets[c + 1] - L->offsets[c];
    a.start[c] = (int32_t)L->offsets[c];
    a.len[c] = (int32_t)len;
    rk[c] = db.add(kv->k[c], len, p.heads, p.d, 128);
    rv[c] = db.add(kv->v[c], len, p.heads, p.d, 128);
  }
  int blocks = 0;
  for (int k = 0; k < a.nq; ++k) {
    const int c = i1 - 1 - k;  // longest chunk first
    const int64_t len = L->offsets[c + 1] - L->offsets[c];
    rq[c - i0] = db.add(q[c - i0], len, p.heads, p.d, 128);
    ro[c - i0] = db.add(o[c - i0], len, p.heads, p.d, 128);
    a.lses[c - i0] = lse[c - i0];
    a.block_base[k] = blocks;
    blocks += (int)((len + 255) / 256);
  }
  a.block_base[a.nq] = blocks;
  if ((s = db.resolve(strm))) return s;
  for (int c = 0; c < kv->n; ++c) {
    a.slots.k[c] = (uint16_t)db.slot(rk[c]);
    a.slots.v[c] = (uint16_t)db.slot(rv[c]);
  }
  for (int k = 0; k < a.nq; ++k) {
    a.qslots[k] = (uint16_t)db.slot(rq[k]);
    a.oslots[k] = (uint16_t)db.slot(ro[k]);
  }
  a.q_slot = a.qslots[0];
  a.o_slot = a.oslots[0];
  a.desc_table = db.table();
  cudaError_t e = launch_fwd_sm100(a, strm);
  if (e == cudaErrorNotSupported) return fail(SPPO_E_UNSUPPORTED, "this request is not implemented by the sm_100a kernels");
  if (e != cudaSuccess) return cuda_fail(e, "sppo_attn_fwd_chunks launch");
  return SPPO_OK;
}

// ---------------------------------------------------------------- backward
sppo_status sppo_attn_bwd(sppo_ctx ctx, const sppo_layout* L, int32_t chunk, const void* q, const sppo_kv_set* kv,
                          const sppo_bwd_args* a, int32_t flags, void* stream) {
  if (!ctx) return fail(SPPO_E_ARG, "ctx is NULL");
  sppo_status s = check_layout(L, chunk);
  if (s) return s;
  if (flags & ~(SPPO_FIRST | SPPO_LAST)) return fail(SPPO_E_ARG, "unknown flags 0x%x", flags);
  const bool first = flags & SPPO_FIRST, last = flags & SPPO_LAST;
  if (!q || !a) return fail(SPPO_E_ARG, "q/args is NULL");
  if (!a->o || !a->lse || !a->dout || !a->delta || !a->dq_acc || !a->dk_acc || !a->dv_acc)
    return fail(SPPO_E_ARG, "bwd args: o/lse/dout/delta/dq_acc/dk_acc/dv_acc must be non-NULL");
  if (last && !a->dq) return fail(SPPO_E_ARG, "dq NULL on LAST");
  if ((a->dk == nullptr) != (a->dv == nullptr)) return fail(SPPO_E_ARG, "dk and dv outputs must both be set or both NULL");
  if (!aligned4(a->lse) || !aligned4(a->delta)) return fail(SPPO_E_ALIGN, "lse/delta not 4B aligned");
  const void* ptrs[] = {q, a->o, a->dout, a->dq_acc, a->dq, a->dk, a->dv};
  for (const void* pp : ptrs)
    if (pp && !aligned16(pp)) return fail(SPPO_E_ALIGN, "bwd tensor not 16B aligned");
  std::lock_guard<std::mutex> lock(ctx->mu);
  const Coverage* cov = nullptr;
  if ((s = lookup_coverage(ctx->cov_bwd, q, chunk, first, &cov))) return s;
  if ((s = check_kv(L, chunk, kv, cov, first, last))) return s;
  int final_slot = -1;
  for (int c = 0; c < kv->n; ++c) {
    if (!a->dk_acc[c] || !a->dv_acc[c]) return fail(SPPO_E_ARG, "dk_acc/dv_acc %d is NULL", c);
    if (!aligned16(a->dk_acc[c]) || !aligned16(a->dv_acc[c])) return fail(SPPO_E_ALIGN, "dk_acc/dv_acc %d misaligned", c);
    if (kv->ids[c] == chunk) final_slot = c;
  }
  if (a->dk && final_slot < 0)
    return fail(SPPO_E_STATE, "dk/dv outputs requested but chunk %d is not in this window", chunk);
  SPPO_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t strm = (cudaStream_t)stream;
  BwdParams p{};
  p.heads = L->heads;
  p.d = L->head_dim;
  p.q_start = (int32_t)L->offsets[chunk];
  p.q_len = (int32_t)(L->offsets[chunk + 1] - L->offsets[chunk]);
  p.scale = L->scale > 0.f ? L->scale : 1.f / sqrtf((float)L->head_dim);
  p.first = first;
  p.last = last;
  p.q = q;
  p.o = a->o;
  p.lse = a->lse;
  p.dout = a->dout;
  p.delta = a->delta;
  p.dq_acc = a->dq_acc;
  p.dq = a->dq;
  p.final_slot = a->dk ? final_slot : -1;
  p.dk_out = a->dk;
  p.dv_out = a->dv;
  p.trace = trace_for(ctx, chunk, true);
  p.trace_life = ctx->trace_life;
  const bool bf16 = L->dtype == SPPO_BF16;
  cudaError_t e = cudaSuccess;
  // host-side preparation first (nothing is enqueued if it fails), then
  // Delta_i / dq_acc = 0 on FIRST (a5), then the main kernel
  auto preprocess = [&]() { return first ? launch_bwd_preprocess(p, bf16, strm) : cudaSuccess; };
  KvWindow w;  // per call: no state shared between contexts or threads
  fill_window(L, kv, &w);
  if (!bf16) {
    KvGradWindow g;
    for (int c = 0; c < kv->n; ++c) {
      g.dk[c] = a->dk_acc[c];
      g.dv[c] = a->dv_acc[c];
    }
    if ((e = preprocess()) != cudaSuccess) return cuda_fail(e, "bwd preprocess");
    e = launch_bwd_simt_f32(p, w, g, strm);
  } else {
    Sm100Bwd sa{};
    sa.p = p;
    sa.n = kv->n;
    DescBlock db;
    db.open(ctx);
    const int rq = db.add(q, p.q_len, p.heads, p.d, 128);
    const int rdo = db.add(a->dout, p.q_len, p.heads, p.d, 128);
    const int rq64 = db.add(q, p.q_len, p.heads, p.d, 64);
    const int rdo64 = db.add(a->dout, p.q_len, p.heads, p.d, 64);
    const int rdq = db.add(a->dq_acc, p.q_len, p.heads, p.d, 128, 4);
    std::vector<int> rk(kv->n), rv(kv->n), rdk(kv->n), rdv(kv->n);
    int pairs = 0;
    for (int c = 0; c < kv->n; ++c) {
      rk[c] = db.add(kv->k[c], w.len[c], p.heads, p.d, 128);
      rv[c] = db.add(kv->v[c], w.len[c], p.heads, p.d, 128);
      rdk[c] = db.add(a->dk_acc[c], w.len[c], p.heads, p.d, 128, 4);
      rdv[c] = db.add(a->dv_acc[c], w.len[c], p.heads, p.d, 128, 4);
      sa.start[c] = w.start[c];
      sa.len[c] = w.len[c];
      sa.pair_base[c] = pairs;
      pairs += (w.len[c] + 255) / 256;
      sa.dk[c] = a->dk_acc[c];
      sa.dv[c] = a->dv_acc[c];
    }
    sa.pair_base[kv->n] = pairs;
    if ((s = db.resolve(strm))) return s;
    sa.q_slot = db.slot(rq);
    sa.do_slot = db.slot(rdo);
    sa.q64_slot = db.slot(rq64);
    sa.do64_slot = db.slot(rdo64);
    sa.dq_slot = db.slot(rdq);
    for (int c = 0; c < kv->n; ++c) {
      sa.slots.k[c] = (uint16_t)db.slot(rk[c]);
      sa.slots.v[c] = (uint16_t)db.slot(rv[c]);
      sa.acc.k[c] = (uint16_t)db.slot(rdk[c]);
      sa.acc.v[c] = (uint16_t)db.slot(rdv[c]);
    }
    sa.desc_table = db.table();
    sa.sched = ctx->sched + (ctx->sched_next++ % kSchedSlots);
    if ((e = preprocess()) != cudaSuccess) return cuda_fail(e, "bwd preprocess");
    if ((e = cudaMemsetAsync(sa.sched, 0, sizeof(int), strm)) != cudaSuccess) return cuda_fail(e, "bwd scheduler reset");
    e = launch_bwd_sm100(sa, strm);
  }
  if (e == cudaErrorNotSupported) return fail(SPPO_E_UNSUPPORTED, "this request is not implemented by the sm_100a kernels");
  if (e != cudaSuccess) return cuda_fail(e, "sppo_attn_bwd launch");
  if (last) {
    e = launch_cast_f32(p.dq_acc, p.dq, (size_t)p.q_len * p.heads * p.d, bf16, strm);  // a7
    if (e != cudaSuccess) return cuda_fail(e, "dq finalize");
  }
  commit_coverage(ctx->cov_bwd, q, chunk, kv, first, last);
  return SPPO_OK;
}

// ---------------------------------------------------------------- host arena + copies
sppo_status sppo_host_alloc(sppo_ctx ctx, size_t bytes, void** host) {
  if (!ctx || !host) return fail(SPPO_E_ARG, "ctx/host is NULL");
  *host = nullptr;
  if (!bytes) return fail(SPPO_E_ARG, "bytes = 0");
  SPPO_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  // NUMA-local to the GPU when its node is known; otherwise (or if the node is
  // out of memory / mbind is refused) a plain portable cudaHostAlloc
  size_t mapped = 0;
  void* p = numa_pinned_alloc(bytes, ctx->numa_node);
  if (p) {
    mapped = bytes;
  } else {
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) return fail(SPPO_E_OOM, "cudaHostAlloc(%zu): %s", bytes, cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  ctx->host_allocs[p] = mapped;
  *host = p;
  return SPPO_OK;
}

sppo_status sppo_host_free(sppo_ctx ctx, void* host) {
  if (!ctx || !host) return fail(SPPO_E_ARG, "ctx/host is NULL");
  std::lock_guard<std::mutex> lock(ctx->mu);
  auto it = ctx->host_allocs.find(host);
  if (it == ctx->host_allocs.end()) return fail(SPPO_E_ARG, "pointer not from sppo_host_alloc");
  const size_t mapped = it->second;
  ctx->host_allocs.erase(it);
  if (mapped) {
    SPPO_CUDA(cudaHostUnregister(host), "cudaHostUnregister");
    if (munmap(host, mapped) != 0) return fail(SPPO_E_ARG, "munmap failed");
  } else {
    SPPO_CUDA(cudaFreeHost(host), "cudaFreeHost");
  }
  return SPPO_OK;
}

sppo_status sppo_ctx_numa_node(sppo_ctx ctx, int32_t* node) {
  if (!ctx || !node) return fail(SPPO_E_ARG, "ctx/node is NULL");
  *node = ctx->numa_node;
  return SPPO_OK;
}

sppo_status sppo_kv_offload(sppo_ctx ctx, int32_t chunk, const void* dev, void* host, size_t bytes, double alpha,
                            void* producer, void* done, size_t* copied) {
  if (!ctx || !dev || !host) return fail(SPPO_E_ARG, "ctx/dev/host is NULL");
  if (chunk < 0) return fail(SPPO_E_ARG, "chunk < 0");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(SPPO_E_ARG, "alpha %g not in [0,1]", alpha);
  const size_t granule = 64 << 10;
  size_t n = (size_t)ceil(alpha * (double)bytes);
  n = (n + granule - 1) / granule * granule;
  if (n > bytes) n = bytes;
  if (copied) *copied = n;
  SPPO_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  SPPO_CUDA(cudaEventRecord(ctx->ev_prod, (cudaStream_t)producer), "offload: record producer");
  SPPO_CUDA(cudaStreamWaitEvent(ctx->d2h, ctx->ev_prod, 0), "offload: wait producer");
  if (n) SPPO_CUDA(cudaMemcpyAsync(host, dev, n, cudaMemcpyDeviceToHost, ctx->d2h), "offload: D2H copy");
  if (done) SPPO_CUDA(cudaEventRecord((cudaEvent_t)done, ctx->d2h), "offload: record done");
  return SPPO_OK;
}

sppo_status sppo_kv_prefetch(sppo_ctx ctx, int32_t chunk, const void* host, void* dev, size_t bytes, void* consumer,
                             void* done, int32_t flags) {
  if (!ctx || !dev || !host) return fail(SPPO_E_ARG, "ctx/dev/host is NULL");
  if (chunk < 0) return fail(SPPO_E_ARG, "chunk < 0");
  if (flags & ~(SPPO_COPY_NO_ORDER | SPPO_COPY_DEFER_WAIT)) return fail(SPPO_E_ARG, "unknown flags 0x%x", flags);
  if ((flags & SPPO_COPY_DEFER_WAIT) && !done) return fail(SPPO_E_ARG, "SPPO_COPY_DEFER_WAIT needs a done event");
  SPPO_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t cons = (cudaStream_t)consumer;
  if (!(flags & SPPO_COPY_NO_ORDER)) {
    SPPO_CUDA(cudaEventRecord(ctx->ev_cons, cons), "prefetch: record consumer");
    SPPO_CUDA(cudaStreamWaitEvent(ctx->h2d, ctx->ev_cons, 0), "prefetch: wait consumer");
  }
  if (bytes) SPPO_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->h2d), "prefetch: H2D copy");
  if (!(flags & SPPO_COPY_DEFER_WAIT)) {
    SPPO_CUDA(cudaEventRecord(ctx->ev_copy, ctx->h2d), "prefetch: record copy");
    SPPO_CUDA(cudaStreamWaitEvent(cons, ctx->ev_copy, 0), "prefetch: consumer wait");
  }
  if (done) SPPO_CUDA(cudaEventRecord((cudaEvent_t)done, ctx->h2d), "prefetch: record done");
  return SPPO_OK;
}

sppo_status sppo_ctx_streams(sppo_ctx ctx, void** d2h, void** h2d) {
  if (!ctx) return fail(SPPO_E_ARG, "ctx is NULL");
  if (d2h) *d2h = ctx->d2h;
  if (h2d) *h2d = ctx->h2d;
  return SPPO_OK;
}

// ---------------------------------------------------------------- plan helpers
sppo_status sppo_partition_equal(int64_t S, int32_t N, int64_t* out) {
  if (!out) return fail(SPPO_E_ARG, "out is NULL");
  if (N < 1 || S < N) return fail(SPPO_E_SHAPE, "need 1 <= N <= S (S=%lld, N=%d)", (long long)S, N);
  const int64_t base = S / N, rem = S % N;
  out[0] = 0;
  for (int32_t i = 0; i < N; ++i) out[i + 1] = out[i] + base + (i < rem ? 1 : 0);
  return SPPO_OK;
}

namespace {
int64_t tri(int64_t x) { return x * (x + 1) / 2; }  // causal pairs of rows 0..x-1

// cost of chunk [a, b): its causal pairs plus `lin` per token (the token-wise
// layer work in pair units; 0 = attention only)
int64_t chunk_cost(int64_t a, int64_t b, int64_t lin) { return tri(b) - tri(a) + lin * (b - a); }

// Largest b in (a, S] with chunk_cost(a, b) <= B (a itself if none).
int64_t greedy_end(int64_t a, int64_t S, int64_t B, int64_t lin = 0) {
  int64_t lo = a, hi = S;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (chunk_cost(a, mid, lin) <= B)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Chunks a greedy cover of [0, S) needs when no chunk may exceed B pairs (INT64_MAX if impossible).
int64_t chunks_needed(int64_t S, int64_t B, int64_t lin = 0) {
  int64_t a = 0, n = 0;
  while (a < S) {
    const int64_t b = greedy_end(a, S, B, lin);
    if (b == a) return INT64_MAX;
    a = b;
    ++n;
  }
  return n;
}
}  // namespace

sppo_status sppo_partition_balanced_lin(int64_t S, int32_t N, int64_t lin, int64_t* out) {
  if (!out) return fail(SPPO_E_ARG, "out is NULL");
  if (N < 1 || S < N || S > (int64_t)INT32_MAX) return fail(SPPO_E_SHAPE, "need 1 <= N <= S < 2^31");
  if (lin < 0 || lin > ((int64_t)1 << 30)) return fail(SPPO_E_ARG, "lin = %lld not in [0, 2^30]", (long long)lin);
  // smallest achievable max-chunk cost B*: binary search on the greedy cover count
  int64_t lo = S + lin, hi = chunk_cost(0, S, lin);  // the last row alone costs S + lin
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (chunks_needed(S, mid, lin) <= N)
      hi = mid;
    else
      lo = mid + 1;
  }
  const int64_t B = lo;
  // lexicographically largest lengths with every chunk <= B and exactly N chunks:
  // each chunk as long as the cost bound allows, leaving >= 1 row per remaining chunk
  out[0] = 0;
  int64_t a = 0;
  for (int32_t i = 0; i < N; ++i) {
    const int64_t remaining = N - i - 1;
    int64_t b = greedy_end(a, S, B, lin);
    if (b > S - remaining) b = S - remaining;
    if (b <= a) return fail(SPPO_E_SHAPE, "balanced partition failed (S=%lld, N=%d)", (long long)S, N);
    out[i + 1] = b;
    a = b;
  }
  if (out[N] != S) return fail(SPPO_E_SHAPE, "balanced partition does not cover S (S=%lld, N=%d)", (long long)S, N);
  return SPPO_OK;
}

sppo_status sppo_partition_balanced(int64_t S, int32_t N, int64_t* out) {
  return sppo_partition_balanced_lin(S, N, 0, out);
}

sppo_status sppo_causal_pairs(const int64_t* off, int32_t N, int64_t* pairs) {
  if (!off || !pairs) return fail(SPPO_E_ARG, "NULL argument");
  if (N < 1) return fail(SPPO_E_SHAPE, "N < 1");
  int64_t total = 0;
  for (int32_t i = 0; i < N; ++i) {
    const int64_t c = off[i], s = off[i + 1] - off[i];
    if (s < 1 || c < 0) return fail(SPPO_E_SHAPE, "offsets not strictly increasing at %d", i);
    total += s * c + s * (s + 1) / 2;
  }
  *pairs = total;
  return SPPO_OK;
}

sppo_status sppo_finalize(sppo_ctx ctx, const float* src, void* dst, size_t n, int32_t dtype, void* stream) {
  if (!ctx || !src || !dst) return fail(SPPO_E_ARG, "NULL argument");
  if (dtype != SPPO_BF16 && dtype != SPPO_FP32) return fail(SPPO_E_ARG, "dtype = %d", dtype);
  if (n % 4) return fail(SPPO_E_SHAPE, "n = %zu is not a multiple of 4", n);
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u)
    return fail(SPPO_E_ALIGN, "src/dst must be 16-byte aligned");
  SPPO_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaError_t e = launch_cast_f32(src, dst, n, dtype == SPPO_BF16, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "sppo_finalize");
  return SPPO_OK;
}

sppo_status sppo_offload_alpha(const double* A, const double* m_threshold, int32_t N, double last, double* alpha) {
  if (!A || !m_threshold || !alpha) return fail(SPPO_E_ARG, "NULL argument");
  if (N < 1) return fail(SPPO_E_SHAPE, "N < 1");
  if (!(last >= 0.0 && last <= 1.0)) return fail(SPPO_E_ARG, "last alpha not in [0,1]");
  for (int32_t i = 0; i < N; ++i)
    if (!(m_threshold[i] >= 0.0)) return fail(SPPO_E_ARG, "m_threshold[%d] < 0", i);
  for (int32_t i = 0; i < N; ++i) {
    if (i == N - 1)
      alpha[i] = last;
    else if (A[i] <= 0.0)
      alpha[i] = 1.0;
    else
      alpha[i] = fmin(1.0, m_threshold[i] / A[i]);
  }
  return SPPO_OK;
}

}  // extern "C"
