// fbf_hostpath.cu -- the host-buffer entry points of the C-ABI
// (include/fourierbf_b200.h): what the drop-in C++ API
// (bilateral_fast(const Image&), bilateral.hpp:109) and bench.py's e2e leg call.
//
//  * fbf_bilateral_fast_host (fp32): pinned or pageable host buffers in and
//    out; calls of >= 1 Mpixel are cut into chunks on two streams so each
//    chunk's H2D / D2H overlaps the neighbouring chunks' kernels; single-launch
//    calls replay a cached CUDA graph.
//  * fbf_bilateral_fast_host_f64 (the reference's Image stores doubles): the
//    same pipeline with the double <-> float conversion done by a persistent
//    host thread pool into pinned staging, chunk by chunk, overlapped with the
//    GPU work of the neighbouring chunks.
//  * fbf_bilateral_fast_host_multi[_f64]: one call over several GPUs of the
//    box, one persistent host worker thread per device, row strips with W halo
//    rows (single image) or whole images (batch) per device; no exchange.
//
// Per calling thread and device: one context (two streams, events, a grow-only
// device buffer, pinned read-back words, the cached graph), freed by
// fbf_release_host_buffers() or when the thread exits.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fbf_common.h"
#include "fbf_device.cuh"
#include "fbf_params.h"
#include "fbf_tuning.h"
#include "fourierbf_b200.h"

namespace fbf {
size_t iir_workspace_bytes(const fbf_geometry* g, int radius);
template <class Tin, class Tout>
int iir_bilateral(const fbf_geometry* g, const fbf_filter* f, const Tin* src, Tout* dst, void* ws, size_t ws_bytes,
                  unsigned long long* d_bad, cudaStream_t st);
}  // namespace fbf

using namespace fbf;

namespace {

constexpr int kMaxChunks = 16;
constexpr int kMaxDevices = 64;

// ------------------------------------------------------------------ contexts

struct HostCtx {
  int dev = -1;
  cudaStream_t st[2] = {nullptr, nullptr};  // chunk streams (copies of one chunk overlap the kernels of the other)
  cudaEvent_t ev[2] = {nullptr, nullptr};   // per stream: the last strip's H2D (halo rows of the next strip)
  cudaEvent_t kdone[2] = {nullptr, nullptr};  // per stream: the last chunk's kernels finished (kernel order = chunk order)
  cudaEvent_t done[kMaxChunks] = {};        // per chunk: its D2H landed (f64 output conversion)
  cudaEvent_t join = nullptr;               // stream 1 back into stream 0
  unsigned long long* h_bad = nullptr;      // pinned: per-chunk collapse indices (graph-capturable read-back)
  char* buf = nullptr;
  size_t cap = 0;
  // the last call's work as a CUDA graph, replayed when the next call is the
  // same (geometry, filter, buffers): one launch instead of ~10 API calls
  std::vector<unsigned char> graph_key;
  cudaGraphExec_t graph = nullptr;

  int open(int d) {
    dev = d;
    for (auto& s : st) FBF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (auto& e : ev) FBF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : kdone) FBF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : done) FBF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    FBF_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    FBF_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_bad), kMaxChunks * sizeof(unsigned long long)));
    return FBF_OK;
  }
  void drop_graph() {
    if (graph) cudaGraphExecDestroy(graph);
    graph = nullptr;
    graph_key.clear();
  }
  int reserve(size_t bytes) {
    if (cap >= bytes) return FBF_OK;
    if (buf) {
      for (auto s : st) cudaStreamSynchronize(s);
      drop_graph();  // it names the old buffer
      cudaFree(buf);
      buf = nullptr;
      cap = 0;
    }
    FBF_CUDA(cudaMalloc(reinterpret_cast<void**>(&buf), bytes));
    cap = bytes;
    return FBF_OK;
  }
  void release() {
    if (dev < 0) return;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    for (auto s : st)
      if (s) cudaStreamSynchronize(s);
    drop_graph();
    if (buf) cudaFree(buf);
    for (auto s : st)
      if (s) cudaStreamDestroy(s);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : kdone)
      if (e) cudaEventDestroy(e);
    for (auto e : done)
      if (e) cudaEventDestroy(e);
    if (join) cudaEventDestroy(join);
    if (h_bad) cudaFreeHost(h_bad);
    if (cur >= 0) cudaSetDevice(cur);
    *this = HostCtx{};
  }
};

// pinned fp32 staging of the f64 entry points (grow-only)
struct Pinned {
  float* p = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes) {
    if (cap >= bytes) return FBF_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    FBF_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), bytes));
    cap = bytes;
    return FBF_OK;
  }
  void release() {
    if (p) cudaFreeHost(p);
    *this = Pinned{};
  }
};

// one context per device for the calling thread, freed at thread exit
struct ThreadState {
  HostCtx ctx[kMaxDevices];
  Pinned pinned;
  ~ThreadState() { release(); }
  void release() {
    for (auto& c : ctx) c.release();
    pinned.release();
  }
};
thread_local ThreadState g_ts;

int host_ctx(size_t bytes, HostCtx*& out) {
  int dev = 0;
  FBF_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(FBF_EUNSUPPORTED, "bilateral_fast: device ordinal out of range");
  HostCtx& c = g_ts.ctx[dev];
  int rc = FBF_OK;
  if (c.dev != dev && (rc = c.open(dev))) return rc;
  if ((rc = c.reserve(bytes))) return rc;
  out = &c;
  return FBF_OK;
}

// ------------------------------------------------------------- thread pool

// A persistent pool for the host-side double <-> float conversions of the f64
// entry points (one process-wide pool; concurrent callers take turns).
// Dispatch is a generation counter: workers spin on it for a while after each
// job before sleeping on the condition variable, and the caller spins on the
// pending count -- a call's successive conversions (and back-to-back calls)
// then start in ~1 us instead of a futex wake-up of every worker per
// conversion, which dominated small calls (c1 e2e_f64, profiles/r02_notes.md).
class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // fn(part, parts) on every worker and the caller; returns when all are done
  void run(const std::function<void(int, int)>& fn) {
    std::lock_guard<std::mutex> call(call_);
    const int parts = size();
    job_ = &fn;
    pending_.store(parts - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(m_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    fn(0, parts);
    while (pending_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
    job_ = nullptr;
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_.store(true);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  Pool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const int n = static_cast<int>(std::max(1u, std::min(hw ? hw : 1u, 16u))) - 1;
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
  }
  void loop(int part) {
    unsigned long long seen = 0;
    for (;;) {
      // spin ~2 ms on the generation counter, then sleep
      const auto t0 = std::chrono::steady_clock::now();
      int it = 0;
      while (gen_.load(std::memory_order_acquire) == seen) {
        if ((++it & 255) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2)) {
          std::unique_lock<std::mutex> lk(m_);
          cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
          break;
        }
      }
      seen = gen_.load(std::memory_order_acquire);
      if (stop_.load()) return;
      (*job_)(part, static_cast<int>(workers_.size()) + 1);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_, m_;
  std::condition_variable cv_;
  const std::function<void(int, int)>* job_ = nullptr;
  std::atomic<int> pending_{0};
  std::atomic<unsigned long long> gen_{0};
  std::atomic<bool> stop_{false};
};

// rows [r0, r1) of each image b in [b0, b1): out (dense, pitch w) <- in (strided)
template <class Tin, class Tout>
void convert_rows(const Tin* in, long long in_bstride, long long in_pitch, Tout* out, long long out_bstride,
                  long long out_pitch, int w, int b0, int b1, int r0, int r1) {
  const long long rows = static_cast<long long>(b1 - b0) * (r1 - r0);
  if (rows <= 0) return;
  Pool::get().run([&](int part, int parts) {
    const long long a = rows * part / parts, e = rows * (part + 1) / parts;
    for (long long k = a; k < e; ++k) {
      const int b = b0 + static_cast<int>(k / (r1 - r0)), r = r0 + static_cast<int>(k % (r1 - r0));
      const Tin* s = in + b * in_bstride + r * in_pitch;
      Tout* d = out + b * out_bstride + r * out_pitch;
      for (int x = 0; x < w; ++x) d[x] = static_cast<Tout>(s[x]);
    }
  });
}

// ------------------------------------------------------------------ chunks

struct Chunk {
  int b0, nb;  // images [b0, b0 + nb)
  int o0, o1;  // output rows (global) [o0, o1)
  int s0, s1;  // source rows (global) [s0, s1) held on the device for this chunk
};

// Calls below kPipelineMinPx run as one launch (CUDA-graph replayed).
// Batches: up to kBatchChunks image chunks, the first and last at 20 %
// weight.  One image: K strips cost ~ a + b/K + c*K (b: the copies a strip
// pipeline hides, c: per-strip prologue rows, launch and tail), fitted on c2 /
// c4 (profiles/r01_notes.md): K = round(sqrt(pixels / kStripPx)) <= 4; the
// first strip's H2D and the last strip's D2H are exposed, so those strips get
// kEdge*Pct % of a middle strip's rows.  Cuts on multiples of 16 rows.
std::vector<Chunk> plan_chunks(const fbf_geometry* g, int W, int variant) {
  std::vector<Chunk> c;
  const double px = static_cast<double>(g->width) * g->out_rows * g->batch;
  if (variant != FBF_VARIANT_FUSED || px < FBF_TUNABLE(HOST_MIN_PX, kPipelineMinPx)) {
    c.push_back({0, g->batch, g->out_row0, g->out_row0 + g->out_rows, g->src_row0, g->src_row0 + g->src_rows});
    return c;
  }
  if (g->batch >= 2) {
    const int k = std::min(g->batch, std::min(static_cast<int>(FBF_TUNABLE(HOST_BATCH_CHUNKS, kBatchChunks)),
                                              kMaxChunks));
    const long long e = k >= 3 ? 20 : 100, wsum = 2 * e + 100LL * (k - 2);
    auto cut = [&](int i) {
      const long long w = i == 0 ? 0 : i == k ? wsum : e + 100LL * (i - 1);
      return static_cast<int>(g->batch * w / wsum);
    };
    for (int i = 0; i < k; ++i) {
      const int b0 = cut(i), b1 = cut(i + 1);
      if (b1 > b0)
        c.push_back({b0, b1 - b0, g->out_row0, g->out_row0 + g->out_rows, g->src_row0, g->src_row0 + g->src_rows});
    }
    return c;
  }
  int best = static_cast<int>(std::lround(std::sqrt(px / FBF_TUNABLE(HOST_STRIP_PX, kStripPx))));
  best = std::max(1, std::min(best, 4));
#ifdef FBF_EXPERIMENTS
  if (const char* force = getenv("FBF_HOST_CHUNKS")) best = std::max(1, std::min(kMaxChunks, atoi(force)));
#endif
  while (best > 1 && g->out_rows / best < 4 * W + 16) --best;
  const long long e_default = px <= 16e6 ? kEdgeSmallPct : kEdgeLargePct;
  const long long e = best >= 3 ? static_cast<long long>(FBF_TUNABLE(HOST_EDGE, e_default)) : 100;
  const long long wsum = 2 * e + 100LL * (best - 2);
  auto cut = [&](int i) {  // cumulative weight of strips [0, i)
    const long long w = i == 0 ? 0 : i == best ? wsum : e + 100LL * (i - 1);
    return g->out_row0 + static_cast<int>(g->out_rows * w / wsum) / 16 * 16;
  };
  for (int i = 0; i < best; ++i) {
    int o0 = cut(i);
    int o1 = i + 1 == best ? g->out_row0 + g->out_rows : cut(i + 1);
    if (i == 0) o0 = g->out_row0;
    if (o1 <= o0) continue;
    const int s0 = std::max(g->src_row0, std::max(0, o0 - W));
    const int s1 = std::min(g->src_row0 + g->src_rows, std::min(g->height, o1 + W));
    c.push_back({0, 1, o0, o1, s0, s1});
  }
  return c;
}

std::string anomaly_message(unsigned long long first_bad, int width, int height) {
  const unsigned long long per = static_cast<unsigned long long>(width) * height;
  const long long inimg = static_cast<long long>(first_bad % per);
  return "bilateral_fast: numerical anomaly, denominator collapsed at pixel (" + std::to_string(inimg % width) +
         ", " + std::to_string(inimg / width) + ")";
}

// ---------------------------------------------------------------- pipeline

// The chunked host pipeline of one call.  Host side of chunk k: `src_host`
// (fp32, the caller's buffer or the pinned staging of the f64 entry) and
// `dst_host`; `before_issue(k)` runs on the calling thread before chunk k's
// work is issued (f64: convert its source rows), `after_done(k)` once chunk
// k's D2H has landed (f64: convert its output rows).
struct Pipeline {
  const fbf_geometry* g;
  const fbf_filter* f;
  int v;
  std::vector<Chunk> chunks;
  long long sb, db;  // device elements per image: source rows, output rows
  HostCtx* ctx = nullptr;
  float* d_src = nullptr;
  float* d_dst = nullptr;
  char* ws0 = nullptr;
  size_t ws_bytes = 0;
  int nws = 1;
  unsigned long long* d_bad = nullptr;

  int setup(const fbf_geometry* g_, const fbf_filter* f_, int v_) {
    g = g_;
    f = f_;
    v = v_;
    chunks = plan_chunks(g, f->radius, v);
    const int K = static_cast<int>(chunks.size());
    if (K > kMaxChunks) return fail(FBF_EINVAL, "bilateral_fast: too many pipeline chunks");
    sb = static_cast<long long>(g->src_rows) * g->width;
    db = static_cast<long long>(g->out_rows) * g->width;
    const size_t src_bytes = static_cast<size_t>(sb) * g->batch * sizeof(float);
    const size_t dst_bytes = static_cast<size_t>(db) * g->batch * sizeof(float);
    ws_bytes = 0;
    for (const Chunk& c : chunks) {
      const fbf_geometry gc = chunk_geometry(c);
      ws_bytes = std::max(ws_bytes, align256(workspace_for(&gc, f, v)));
    }
    nws = K > 1 ? 2 : 1;
    const size_t total = align256(src_bytes) + align256(dst_bytes) + nws * ws_bytes + align256(K * 8) + 256;
    int rc = host_ctx(total, ctx);
    if (rc) return rc;
    d_src = reinterpret_cast<float*>(ctx->buf);
    d_dst = reinterpret_cast<float*>(ctx->buf + align256(src_bytes));
    ws0 = ctx->buf + align256(src_bytes) + align256(dst_bytes);
    d_bad = reinterpret_cast<unsigned long long*>(ws0 + nws * ws_bytes);
    return FBF_OK;
  }
  fbf_geometry chunk_geometry(const Chunk& c) const {
    fbf_geometry gc = *g;
    gc.batch = c.nb;
    gc.src_row0 = c.s0;
    gc.src_rows = c.s1 - c.s0;
    gc.out_row0 = c.o0;
    gc.out_rows = c.o1 - c.o0;
    gc.src_pitch = g->width;
    gc.dst_pitch = g->width;
    gc.src_bstride = sb;
    gc.dst_bstride = db;
    return gc;
  }
  // first source row chunk k copies (row strips: the rows no earlier strip copied)
  int copy_row0(int k) const {
    const Chunk& c = chunks[k];
    if (g->batch >= 2 || chunks.size() == 1 || k == 0) return c.s0;
    return std::max(c.s0, chunks[k - 1].s1);
  }
  int issue_head() {
    const int K = static_cast<int>(chunks.size());
    cudaError_t e = cudaMemsetAsync(d_bad, 0xFF, K * sizeof(unsigned long long), ctx->st[0]);
    if (e == cudaSuccess && K > 1) e = cudaEventRecord(ctx->ev[1], ctx->st[0]);
    if (e == cudaSuccess && K > 1) e = cudaStreamWaitEvent(ctx->st[1], ctx->ev[1], 0);
    return e == cudaSuccess ? FBF_OK : cuda_fail(e, "memset");
  }
  // H2D -> kernels -> D2H of chunk k on stream k & 1
  int issue_chunk(int k, const float* src, long long src_bstride, long long src_pitch, float* dst,
                  long long dst_bstride, long long dst_pitch, bool record_done) {
    const int K = static_cast<int>(chunks.size());
    const Chunk& c = chunks[k];
    cudaStream_t st = ctx->st[k & 1];
    cudaError_t e = cudaSuccess;
    const int r0 = copy_row0(k);
    // images stacked without gaps (whole rows, bstride = rows * pitch): one 2-D copy
    const bool src_stacked = r0 == g->src_row0 && c.s1 == g->src_row0 + g->src_rows &&
                             src_bstride == static_cast<long long>(g->src_rows) * src_pitch;
    for (int b = c.b0; b < c.b0 + c.nb && r0 < c.s1; b += src_stacked ? c.nb : 1) {
      e = cudaMemcpy2DAsync(d_src + b * sb + static_cast<long long>(r0 - g->src_row0) * g->width,
                            g->width * sizeof(float),
                            src + b * src_bstride + static_cast<long long>(r0 - g->src_row0) * src_pitch,
                            src_pitch * sizeof(float), g->width * sizeof(float),
                            src_stacked ? static_cast<size_t>(c.nb) * g->src_rows : c.s1 - r0,
                            cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "H2D");
    }
    if (g->batch < 2 && K > 1) {
      // the strip's upper halo rows came with the previous strip, on the other stream
      if (k > 0 && c.s0 < chunks[k - 1].s1) e = cudaStreamWaitEvent(st, ctx->ev[(k - 1) & 1], 0);
      if (e == cudaSuccess) e = cudaEventRecord(ctx->ev[k & 1], st);
      if (e != cudaSuccess) return cuda_fail(e, "event");
    }
    // Kernels run in chunk order: chunk k's start behind chunk k-1's last
    // kernel.  Every fused kernel fills the GPU, so nothing is lost; without
    // the edge, chunk k's fused kernel can take the SMs ahead of chunk k-1's
    // closing n = 0 / finish kernel (ready at the same moment on the other
    // stream) and hold back that chunk's D2H, and the H2D queued behind it, for
    // a whole kernel (c2 e2e 1.34 -> 1.54 ms when that happened).
    if (K > 1 && k > 0 && (e = cudaStreamWaitEvent(st, ctx->kdone[(k - 1) & 1], 0)) != cudaSuccess)
      return cuda_fail(e, "event");
    const fbf_geometry gc = chunk_geometry(c);
    const int rc = fbf_bilateral_fast_device(&gc, f, d_src + c.b0 * sb + static_cast<long long>(c.s0 - g->src_row0) * g->width,
                                             d_dst + c.b0 * db + static_cast<long long>(c.o0 - g->out_row0) * g->width,
                                             ws0 + (k & 1) * (nws > 1 ? ws_bytes : 0), ws_bytes, d_bad + k, v, st);
    if (rc != FBF_OK) return rc;
    if (K > 1 && (e = cudaEventRecord(ctx->kdone[k & 1], st)) != cudaSuccess) return cuda_fail(e, "event");
    const bool dst_stacked = c.o0 == g->out_row0 && c.o1 == g->out_row0 + g->out_rows &&
                             dst_bstride == static_cast<long long>(g->out_rows) * dst_pitch;
    for (int b = c.b0; b < c.b0 + c.nb; b += dst_stacked ? c.nb : 1) {
      e = cudaMemcpy2DAsync(dst + b * dst_bstride + static_cast<long long>(c.o0 - g->out_row0) * dst_pitch,
                            dst_pitch * sizeof(float),
                            d_dst + b * db + static_cast<long long>(c.o0 - g->out_row0) * g->width,
                            g->width * sizeof(float), g->width * sizeof(float),
                            dst_stacked ? static_cast<size_t>(c.nb) * g->out_rows : c.o1 - c.o0,
                            cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_fail(e, "D2H");
    }
    if (record_done && (e = cudaEventRecord(ctx->done[k], st)) != cudaSuccess) return cuda_fail(e, "event");
    return FBF_OK;
  }
  int issue_tail() {
    const int K = static_cast<int>(chunks.size());
    cudaError_t e = cudaSuccess;
    if (K > 1) {
      e = cudaEventRecord(ctx->join, ctx->st[1]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->st[0], ctx->join, 0);
      if (e != cudaSuccess) return cuda_fail(e, "join");
    }
    e = cudaMemcpyAsync(ctx->h_bad, d_bad, K * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->st[0]);
    return e == cudaSuccess ? FBF_OK : cuda_fail(e, "D2H");
  }
  // after the stream sync: the reference's anomaly (first collapsed pixel)
  int verdict(int out, long long* bad_index) {
    cudaError_t e = cudaStreamSynchronize(ctx->st[0]);
    if (out == FBF_OK && e != cudaSuccess) out = cuda_fail(e, "sync");
    if (out != FBF_OK) {
      cudaStreamSynchronize(ctx->st[1]);
      return out;
    }
    // chunk-local image index -> the call's (the kernels number images from 0 per launch)
    const unsigned long long per_img = static_cast<unsigned long long>(g->width) * g->height;
    unsigned long long first_bad = ~0ULL;
    for (size_t k = 0; k < chunks.size(); ++k)
      if (ctx->h_bad[k] != ~0ULL)
        first_bad = std::min(first_bad, ctx->h_bad[k] + static_cast<unsigned long long>(chunks[k].b0) * per_img);
    if (first_bad != ~0ULL) {
      if (bad_index) *bad_index = static_cast<long long>(first_bad);
      return fail(FBF_EANOMALY, anomaly_message(first_bad, g->width, g->height));
    }
    return FBF_OK;
  }
};

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  return ok;
}

// Host-buffer entry of the recursive backend: whole images, fp64 inside,
// T-typed host buffers in and out (the f64 entry keeps the reference's doubles).
template <class T>
int iir_host(const fbf_geometry* g, const fbf_filter* f, const T* src, T* dst, long long* bad_index) {
  fbf_geometry gd = *g;
  gd.src_pitch = g->width;
  gd.dst_pitch = g->width;
  gd.src_bstride = static_cast<long long>(g->src_rows) * g->width;
  gd.dst_bstride = static_cast<long long>(g->out_rows) * g->width;
  const size_t src_bytes = static_cast<size_t>(gd.src_bstride) * g->batch * sizeof(T);
  const size_t dst_bytes = static_cast<size_t>(gd.dst_bstride) * g->batch * sizeof(T);
  const size_t ws_bytes = iir_workspace_bytes(g, f->radius);
  HostCtx* ctx = nullptr;
  int rc = host_ctx(align256(src_bytes) + align256(dst_bytes) + ws_bytes + 256, ctx);
  if (rc) return rc;
  cudaStream_t st = ctx->st[0];
  T* d_src = reinterpret_cast<T*>(ctx->buf);
  T* d_dst = reinterpret_cast<T*>(ctx->buf + align256(src_bytes));
  char* ws = ctx->buf + align256(src_bytes) + align256(dst_bytes);
  unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(ws + ws_bytes);
  for (int b = 0; b < g->batch; ++b)
    FBF_CUDA(cudaMemcpy2DAsync(d_src + b * gd.src_bstride, g->width * sizeof(T), src + b * g->src_bstride,
                               g->src_pitch * sizeof(T), g->width * sizeof(T), g->src_rows, cudaMemcpyHostToDevice,
                               st));
  FBF_CUDA(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), st));
  rc = iir_bilateral<T, T>(&gd, f, d_src, d_dst, ws, ws_bytes, d_bad, st);
  if (rc) {
    cudaStreamSynchronize(st);
    return rc;
  }
  for (int b = 0; b < g->batch; ++b)
    FBF_CUDA(cudaMemcpy2DAsync(dst + b * g->dst_bstride, g->dst_pitch * sizeof(T), d_dst + b * gd.dst_bstride,
                               g->width * sizeof(T), g->width * sizeof(T), g->out_rows, cudaMemcpyDeviceToHost, st));
  FBF_CUDA(cudaMemcpyAsync(ctx->h_bad, d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  FBF_CUDA(cudaStreamSynchronize(st));
  const unsigned long long bad = ctx->h_bad[0];
  if (bad != ~0ULL) {
    if (bad_index) *bad_index = static_cast<long long>(bad);
    return fail(FBF_EANOMALY, anomaly_message(bad, g->width, g->height));
  }
  return FBF_OK;
}

int resolve_variant(const fbf_filter* f, int variant) {
  int v = variant;
  if (v == FBF_VARIANT_RECURSIVE) v = FBF_VARIANT_FUSED;  // box windows and sigma < 2 stay direct (spatial.hpp:102-104)
  if (v == FBF_VARIANT_FUSED && !fused_applies(f)) v = FBF_VARIANT_NAIVE;
  return v;
}

// ------------------------------------------------------------ multi-device

// One persistent worker thread per device: its thread-local contexts (streams,
// buffers, cached graphs) stay warm across calls.
class DeviceWorker {
 public:
  explicit DeviceWorker(int dev) : dev_(dev), t_([this] { loop(); }) {}
  ~DeviceWorker() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    t_.join();
  }
  std::future<std::pair<int, std::string>> submit(std::function<int()> job) {
    auto task = std::make_shared<std::packaged_task<std::pair<int, std::string>()>>([job] {
      const int rc = job();
      return std::make_pair(rc, rc == FBF_OK ? std::string() : std::string(fbf_last_error()));
    });
    auto fut = task->get_future();
    {
      std::lock_guard<std::mutex> lk(m_);
      q_.push_back([task] { (*task)(); });
    }
    cv_.notify_all();
    return fut;
  }

 private:
  void loop() {
    cudaSetDevice(dev_);
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty()) return;
        job = std::move(q_.front());
        q_.erase(q_.begin());
      }
      job();
    }
  }
  int dev_;
  std::mutex m_;
  std::condition_variable cv_;
  std::vector<std::function<void()>> q_;
  bool stop_ = false;
  std::thread t_;
};

DeviceWorker& worker_for(int dev) {
  static std::mutex m;
  static std::unique_ptr<DeviceWorker> w[kMaxDevices];
  std::lock_guard<std::mutex> lk(m);
  if (!w[dev]) w[dev] = std::make_unique<DeviceWorker>(dev);
  return *w[dev];
}

// The call split over `ndev` devices: a batch by whole images, one image by
// row strips cut on multiples of 16 rows (the column-pass block: every strip
// reproduces the single-GPU bits), each strip holding its W halo rows.
template <class T, class Entry>
int multi_device(const fbf_geometry* g, const fbf_filter* f, const T* src, T* dst, int variant, long long* bad_index,
                 const int* devices, int ndev, Entry entry) {
  int rc = check_call(g, f);
  if (rc) return rc;
  if (!devices || ndev < 1 || ndev > kMaxDevices) return fail(FBF_EINVAL, "bilateral_fast: no devices");
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= kMaxDevices) return fail(FBF_EINVAL, "bilateral_fast: bad device ordinal");
  struct Part {
    fbf_geometry g;
    const T* src;
    T* dst;
    unsigned long long b0;
  };
  std::vector<Part> parts;
  if (g->batch >= ndev || g->batch > 1) {
    for (int i = 0; i < ndev; ++i) {
      const int b0 = static_cast<int>(static_cast<long long>(g->batch) * i / ndev);
      const int b1 = static_cast<int>(static_cast<long long>(g->batch) * (i + 1) / ndev);
      if (b1 <= b0) continue;
      Part p{*g, src + b0 * g->src_bstride, dst + b0 * g->dst_bstride, static_cast<unsigned long long>(b0)};
      p.g.batch = b1 - b0;
      parts.push_back(p);
    }
  } else {
    const int W = f->radius;
    auto cut = [&](int i) {
      if (i == 0) return g->out_row0;
      if (i == ndev) return g->out_row0 + g->out_rows;
      return g->out_row0 + static_cast<int>(static_cast<long long>(g->out_rows) * i / ndev) / 16 * 16;
    };
    for (int i = 0; i < ndev; ++i) {
      const int o0 = cut(i), o1 = cut(i + 1);
      if (o1 <= o0) continue;
      // mirrored rows the strip's outputs read (its W halo rows; mirror only at the global edges)
      int lo = g->height, hi = -1;
      auto visit = [&](int y) {
        for (int k = -W; k <= W; ++k) {
          const int s = mirror_index(y + k, g->height);
          lo = std::min(lo, s);
          hi = std::max(hi, s);
        }
      };
      for (int y = o0; y < std::min(o1, o0 + 2 * W + 1); ++y) visit(y);
      for (int y = std::max(o0, o1 - 2 * W - 1); y < o1; ++y) visit(y);
      Part p{*g, src + static_cast<long long>(lo - g->src_row0) * g->src_pitch,
             dst + static_cast<long long>(o0 - g->out_row0) * g->dst_pitch, 0ull};
      p.g.src_row0 = lo;
      p.g.src_rows = hi + 1 - lo;
      p.g.out_row0 = o0;
      p.g.out_rows = o1 - o0;
      parts.push_back(p);
    }
  }
  std::vector<std::future<std::pair<int, std::string>>> futs;
  std::vector<long long> bads(parts.size(), -1);
  for (size_t i = 0; i < parts.size(); ++i) {
    const Part* p = &parts[i];
    long long* b = &bads[i];
    futs.push_back(worker_for(devices[i % ndev]).submit([p, f, variant, b, entry] {
      return entry(&p->g, f, p->src, p->dst, variant, b);
    }));
  }
  int out = FBF_OK;
  std::string msg;
  unsigned long long first_bad = ~0ULL;
  for (size_t i = 0; i < futs.size(); ++i) {
    const auto r = futs[i].get();
    if (r.first == FBF_EANOMALY && bads[i] >= 0) {
      first_bad = std::min(first_bad, static_cast<unsigned long long>(bads[i]) +
                                          parts[i].b0 * static_cast<unsigned long long>(g->width) * g->height);
    } else if (r.first != FBF_OK && out == FBF_OK) {
      out = r.first;
      msg = r.second;
    }
  }
  if (out != FBF_OK) return fail(out, msg);
  if (first_bad != ~0ULL) {
    if (bad_index) *bad_index = static_cast<long long>(first_bad);
    return fail(FBF_EANOMALY, anomaly_message(first_bad, g->width, g->height));
  }
  return FBF_OK;
}

}  // namespace

extern "C" {

int fbf_bilateral_fast_host(const fbf_geometry* g, const fbf_filter* f, const float* src, float* dst, int variant,
                            long long* bad_index) {
  int rc = check_call(g, f);
  if (rc) return rc;
  if (variant == FBF_VARIANT_RECURSIVE && recursive_applies(f)) return iir_host<float>(g, f, src, dst, bad_index);
  Pipeline pl;
  if ((rc = pl.setup(g, f, resolve_variant(f, variant)))) return rc;
  const int K = static_cast<int>(pl.chunks.size());
  auto issue = [&]() -> int {
    int r = pl.issue_head();
    for (int k = 0; r == FBF_OK && k < K; ++k)
      r = pl.issue_chunk(k, src, g->src_bstride, g->src_pitch, dst, g->dst_bstride, g->dst_pitch, false);
    return r == FBF_OK ? pl.issue_tail() : r;
  };
  HostCtx* ctx = pl.ctx;
  // graph replay key: everything the issued work depends on
  std::vector<unsigned char> key;
  auto put = [&](const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    key.insert(key.end(), c, c + n);
  };
  put(g, sizeof(*g));
  put(&f->kind, sizeof(f->kind));
  put(&f->radius, sizeof(f->radius));
  put(&f->w0, sizeof(f->w0));
  put(&f->N, sizeof(f->N));
  put(&f->omega, sizeof(f->omega));
  put(&f->max_pointwise_error, sizeof(f->max_pointwise_error));
  put(&f->check_epsilon, sizeof(f->check_epsilon));
  put(f->d, (f->N + 1) * sizeof(double));
  put(f->profile, (2 * f->radius + 1) * sizeof(double));
  put(&pl.v, sizeof(pl.v));
  put(&src, sizeof(src));
  put(&dst, sizeof(dst));
  put(&ctx->buf, sizeof(ctx->buf));
  // graphs pay off for single-launch calls (c1 / c3 e2e +13-15 %); replaying the
  // two-stream pipeline measured slower than issuing it (c2 -5 %)
  const bool graphs = K == 1;
  int out = FBF_OK;
  if (graphs && ctx->graph && key == ctx->graph_key) {
    const cudaError_t e = cudaGraphLaunch(ctx->graph, ctx->st[0]);
    out = e == cudaSuccess ? FBF_OK : cuda_fail(e, "graph launch");
  } else if (graphs && is_pinned(src) && is_pinned(dst)) {
    // record this call as a graph (pageable host buffers cannot be captured)
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(ctx->st[0], cudaStreamCaptureModeThreadLocal);
    out = e == cudaSuccess ? issue() : cuda_fail(e, "capture");
    if (e == cudaSuccess) e = cudaStreamEndCapture(ctx->st[0], &graph);
    cudaGraphExec_t exec = nullptr;
    if (out == FBF_OK && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (out == FBF_OK && e == cudaSuccess) {
      ctx->drop_graph();
      ctx->graph = exec;
      ctx->graph_key = std::move(key);
      e = cudaGraphLaunch(exec, ctx->st[0]);
      out = e == cudaSuccess ? FBF_OK : cuda_fail(e, "graph launch");
    } else {  // capture not possible here: issue directly
      if (exec) cudaGraphExecDestroy(exec);
      cudaGetLastError();
      out = issue();
    }
  } else {
    out = issue();
  }
  return pl.verdict(out, bad_index);
}

// fp64 host buffers (the reference's Image): the fp32 pipeline with the
// conversions on the host thread pool into pinned staging, overlapped with the
// GPU: chunk k+1's input conversion runs while chunk k is on the device, and
// chunk k's output conversion while the later chunks are.
int fbf_bilateral_fast_host_f64(const fbf_geometry* g, const fbf_filter* f, const double* src, double* dst,
                                int variant, long long* bad_index) {
  int rc = check_call(g, f);
  if (rc) return rc;
  if (variant == FBF_VARIANT_RECURSIVE && recursive_applies(f)) return iir_host<double>(g, f, src, dst, bad_index);
  Pipeline pl;
  if ((rc = pl.setup(g, f, resolve_variant(f, variant)))) return rc;
  const int K = static_cast<int>(pl.chunks.size());
  // pinned fp32 staging: dense source rows of the call, then its output rows
  const long long ns = pl.sb * g->batch, nd = pl.db * g->batch;
  if ((rc = g_ts.pinned.reserve(static_cast<size_t>(ns + nd) * sizeof(float)))) return rc;
  float* hs = g_ts.pinned.p;
  float* hd = hs + ns;
  rc = pl.issue_head();
  for (int k = 0; rc == FBF_OK && k < K; ++k) {
    const Chunk& c = pl.chunks[k];
    const int r0 = pl.copy_row0(k);
    convert_rows(src + static_cast<long long>(r0 - g->src_row0) * g->src_pitch, g->src_bstride, g->src_pitch,
                 hs + static_cast<long long>(r0 - g->src_row0) * g->width, pl.sb, g->width, g->width, c.b0,
                 c.b0 + c.nb, 0, c.s1 - r0);
    rc = pl.issue_chunk(k, hs, pl.sb, g->width, hd, pl.db, g->width, true);
  }
  if (rc == FBF_OK) rc = pl.issue_tail();
  for (int k = 0; rc == FBF_OK && k < K; ++k) {
    const cudaError_t e = cudaEventSynchronize(pl.ctx->done[k]);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "sync");
      break;
    }
    const Chunk& c = pl.chunks[k];
    const long long o = static_cast<long long>(c.o0 - g->out_row0);
    convert_rows(hd + o * g->width, pl.db, g->width, dst + o * g->dst_pitch, g->dst_bstride, g->dst_pitch, g->width,
                 c.b0, c.b0 + c.nb, 0, c.o1 - c.o0);
  }
  return pl.verdict(rc, bad_index);
}

int fbf_bilateral_fast_host_multi(const fbf_geometry* g, const fbf_filter* f, const float* src, float* dst,
                                  int variant, long long* bad_index, const int* devices, int ndevices) {
  return multi_device<float>(g, f, src, dst, variant, bad_index, devices, ndevices, fbf_bilateral_fast_host);
}

int fbf_bilateral_fast_host_multi_f64(const fbf_geometry* g, const fbf_filter* f, const double* src, double* dst,
                                      int variant, long long* bad_index, const int* devices, int ndevices) {
  return multi_device<double>(g, f, src, dst, variant, bad_index, devices, ndevices, fbf_bilateral_fast_host_f64);
}

void fbf_release_host_buffers(void) { g_ts.release(); }

int fbf_convolve_host_f64(int width, int height, const double* profile, int radius, const double* src,
                          double* dst) {
  if (width <= 0 || height <= 0) return fail(FBF_EINVAL, "convolve: empty plane");
  const size_t n = static_cast<size_t>(width) * height;
  const size_t ws = fbf_convolve_workspace_bytes(width, height, radius);
  HostCtx* ctx = nullptr;
  int rc = host_ctx(2 * align256(n * sizeof(double)) + ws, ctx);
  if (rc) return rc;
  cudaStream_t st = ctx->st[0];
  double* ds = reinterpret_cast<double*>(ctx->buf);
  double* dd = reinterpret_cast<double*>(ctx->buf + align256(n * sizeof(double)));
  void* w = ctx->buf + 2 * align256(n * sizeof(double));
  cudaError_t e = cudaMemcpyAsync(ds, src, n * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "convolve H2D");
  rc = fbf_convolve_device_f64(width, height, profile, radius, ds, dd, w, ws, st);
  if (rc == FBF_OK) {
    e = cudaMemcpyAsync(dst, dd, n * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "convolve D2H");
  }
  cudaStreamSynchronize(st);
  return rc;
}

}  // extern "C"
