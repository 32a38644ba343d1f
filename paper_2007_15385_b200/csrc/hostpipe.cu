// hostpipe.cu -- the host-buffer side of the C-ABI: vpipg_test_host_multi,
// vpipg_test_host, vpipg_test_gather_host and vpipg_release_staging.
//
// Points that live in host memory cross PCIe once per call in chunks, on three
// streams, through a per-device staging area kept between calls. Pinned
// buffers are DMA'd directly; pageable ones (a std::vector behind the vpip::
// shim, a numpy array) are copied into pinned bounce slots by a small host
// thread pool while earlier chunks are on the link. Every point test still
// runs in a device kernel (capi::dispatch / launch_gather).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "capi_internal.h"

using namespace vpipg;
using namespace vpipg::capi;

extern "C" {

namespace {

// Per-device staging for the host-buffer path: kSlots chunk slots (points,
// mask words, mask bytes, counts) and their streams, allocated on first use,
// grown on demand and kept for the life of the process (vpipg_release_staging
// frees them), so a steady stream of host batches pays no allocation, stream
// creation or pool trimming per call. Calls on one device serialise on its
// mutex -- they share the PCIe link anyway.
constexpr int kSlots = 3;
constexpr uint64_t kChunk = uint64_t(1) << 24;  // 16 Mi points, 32-aligned

struct Staging {
  std::mutex mu;
  cudaStream_t st[kSlots] = {};
  char* buf[kSlots] = {};
  size_t cap = 0;  // bytes per slot
  // pageable-host path: pinned bounce buffers (points in, mask words out) and
  // one completion event per slot
  char* hin[kSlots] = {};
  char* hout[kSlots] = {};
  size_t hcap_in = 0, hcap_out = 0;
  cudaEvent_t ev[kSlots] = {};
};

}  // namespace
}  // extern "C"

namespace {

// A small persistent host thread pool for the pageable-buffer copies: one
// std::thread per hardware thread (at most 16). parallel_for publishes a job
// (function, item count, counters); the caller and any worker that wakes in
// time take items until none are left, and the caller returns as soon as every
// item is done -- a worker that wakes late finds the job exhausted and goes
// back to sleep, so no call waits for thread wake-ups.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  template <class F>
  void parallel_for(int n, F&& fn) {
    if (n <= 0) return;
    if (workers_.empty() || n == 1) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    auto job = std::make_shared<Job>();
    job->fn = [&fn](int i) { fn(i); };
    job->n = n;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = job;
      ++gen_;
    }
    cv_.notify_all();
    run(*job);
    std::unique_lock<std::mutex> lk(job->mu);
    job->cv.wait(lk, [&] { return job->done.load() == job->n; });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  struct Job {
    std::function<void(int)> fn;
    int n = 0;
    std::atomic<int> next{0}, done{0};
    std::mutex mu;
    std::condition_variable cv;
  };
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned n = std::min(16u, hw);
    for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  static void run(Job& job) {
    for (int i = job.next.fetch_add(1); i < job.n; i = job.next.fetch_add(1)) {
      job.fn(i);
      if (job.done.fetch_add(1) + 1 == job.n) {
        std::lock_guard<std::mutex> lk(job.mu);
        job.cv.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Job> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
      }
      if (job) run(*job);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// memcpy split into 256 KiB pieces over the pool
void pool_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = size_t(1) << 18;
  const int pieces = static_cast<int>((bytes + kPiece - 1) / kPiece);
  HostPool::get().parallel_for(pieces, [&](int i) {
    const size_t o = size_t(i) * kPiece;
    std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                std::min(kPiece, bytes - o));
  });
}

// mask words (bit j of the stream = point j) -> one byte per point
void pool_expand_bits(uint8_t* dst, const uint32_t* words, uint64_t m) {
  static const std::array<uint64_t, 256> lut = [] {
    std::array<uint64_t, 256> t{};
    for (int b = 0; b < 256; ++b)
      for (int k = 0; k < 8; ++k) t[b] |= uint64_t((b >> k) & 1) << (8 * k);
    return t;
  }();
  const uint8_t* src = reinterpret_cast<const uint8_t*>(words);
  constexpr uint64_t kPiece = uint64_t(1) << 16;  // points per piece (multiple of 8)
  const int pieces = static_cast<int>((m + kPiece - 1) / kPiece);
  HostPool::get().parallel_for(pieces, [&](int i) {
    const uint64_t lo = uint64_t(i) * kPiece, hi = std::min(m, lo + kPiece);
    uint64_t j = lo;
    for (; j + 8 <= hi; j += 8) {
      const uint64_t v = lut[src[j / 8]];
      std::memcpy(dst + j, &v, 8);
    }
    for (; j < hi; ++j) dst[j] = (src[j / 8] >> (j % 8)) & 1u;
  });
}

bool host_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {
namespace {

Staging& staging(int device) {
  static Staging s[64];
  return s[device];
}

struct SlotView {
  void* x;
  void* y;
  uint32_t* w[3];
  uint8_t* b[3];
  unsigned long long* c;
};

size_t slot_bytes(uint64_t chunk, size_t elt, bool bytes) {
  const uint64_t words = (chunk + 31) / 32;
  return 2 * align256(chunk * elt) + 3 * align256(words * 4) + (bytes ? 3 * align256(chunk) : 0) + 256;
}

SlotView slot_view(char* b, uint64_t chunk, size_t elt, bool bytes) {
  SlotView v{};
  size_t off = 0;
  auto take = [&](size_t n) { char* q = b + off; off += align256(n); return q; };
  v.x = take(chunk * elt);
  v.y = take(chunk * elt);
  for (auto& w : v.w) w = reinterpret_cast<uint32_t*>(take((chunk + 31) / 32 * 4));
  for (auto& q : v.b) q = bytes ? reinterpret_cast<uint8_t*>(take(chunk)) : nullptr;
  v.c = reinterpret_cast<unsigned long long*>(take(24));
  return v;
}

// Caller holds st.mu and the device guard.
int staging_reserve(Staging& st, size_t need) {
  if (!st.st[0])
    for (auto& s : st.st) VPIPG_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  if (need <= st.cap) return kOk;
  for (auto& b : st.buf) {
    if (b) cudaFree(b);
    b = nullptr;
  }
  st.cap = 0;
  for (auto& b : st.buf) VPIPG_TRY(cudaMalloc(&b, need));
  st.cap = need;
  return kOk;
}

// Caller holds st.mu and the device guard.
int host_reserve(Staging& st, size_t in_bytes, size_t out_bytes) {
  for (auto& e : st.ev)
    if (!e) VPIPG_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (in_bytes > st.hcap_in) {
    for (auto& b : st.hin) {
      if (b) cudaFreeHost(b);
      b = nullptr;
    }
    st.hcap_in = 0;
    for (auto& b : st.hin) VPIPG_TRY(cudaMallocHost(&b, in_bytes));
    st.hcap_in = in_bytes;
  }
  if (out_bytes > st.hcap_out) {
    for (auto& b : st.hout) {
      if (b) cudaFreeHost(b);
      b = nullptr;
    }
    st.hcap_out = 0;
    for (auto& b : st.hout) VPIPG_TRY(cudaMallocHost(&b, out_bytes));
    st.hcap_out = out_bytes;
  }
  return kOk;
}

// pageable chunks: about 1/8 of the batch (so even a 1 Mi-point call overlaps
// its bounce copies with the link), 64 Ki .. 2 Mi points, 32-aligned
uint64_t host_chunk(uint64_t m) {
  uint64_t c = (m / 8 + 31) & ~uint64_t(31);
  return std::min<uint64_t>(std::max<uint64_t>(c, uint64_t(1) << 16), uint64_t(1) << 21);
}

// Device slot of the generic host pipeline: up to 3 input arrays, the mask
// words of the 3 engines and the 3 counters.
struct PipeSlot {
  void* in[3];
  uint32_t* w[3];
  unsigned long long* c;
};

size_t pipe_slot_bytes(uint64_t chunk, const size_t* elt, int nin) {
  size_t b = 3 * align256((chunk + 31) / 32 * 4) + 256;
  for (int k = 0; k < nin; ++k) b += align256(chunk * elt[k]);
  return b;
}

PipeSlot pipe_slot_view(char* base, uint64_t chunk, const size_t* elt, int nin) {
  PipeSlot v{};
  size_t off = 0;
  auto take = [&](size_t n) { char* q = base + off; off += align256(n); return q; };
  for (int k = 0; k < nin; ++k) v.in[k] = take(chunk * elt[k]);
  for (auto& w : v.w) w = reinterpret_cast<uint32_t*>(take((chunk + 31) / 32 * 4));
  v.c = reinterpret_cast<unsigned long long*>(take(24));
  return v;
}

// Launches engine e on one chunk: device inputs, length, mask words (may be
// NULL), counter; returns a library code.
using ChunkLaunch = std::function<int(int e, void* const* din, uint64_t len, uint32_t* dw,
                                      unsigned long long* dc, cudaStream_t s)>;

// The host-buffer pipeline for pageable memory (a std::vector behind the vpip::
// shim, a numpy array): the pool copies each chunk's inputs into a pinned
// bounce slot while the GPU works on the previous chunks, the copy engine
// moves it at link rate, the engines write mask WORDS (1/8 of the byte mask
// on the link), and the pool copies / expands them into the caller's words or
// bytes once that slot's event fires. Pinned inputs skip the bounce copy.
// Caller holds st.mu and the device guard.
int host_pipeline(Staging& st, const void* const* hin, const size_t* elt, int nin, uint64_t m,
                  const int* eng, int ne, uint32_t* const* mask_words, uint8_t* const* mask_bytes,
                  uint64_t* inside, const ChunkLaunch& launch) {
  bool in_pinned = true;
  for (int k = 0; k < nin; ++k) in_pinned = in_pinned && host_pinned(hin[k]);
  // pinned word outputs and no byte outputs: the D2H lands in the caller's
  // words directly and, with pinned inputs too, nothing waits until the end
  bool direct_out = true;
  for (int k = 0; k < ne; ++k) {
    const int e = eng[k];
    if (mask_bytes && mask_bytes[e]) direct_out = false;
    if (mask_words && mask_words[e] && !host_pinned(mask_words[e])) direct_out = false;
  }
  const bool waits = !(in_pinned && direct_out);
  // nothing to wait for: larger chunks (m/8, 1-16 Mi) straight to the copy
  // engine; otherwise m/8 in 64 Ki-2 Mi so copy-in / copy-out overlap finely
  const uint64_t want_chunk =
      waits ? host_chunk(m)
            : std::min<uint64_t>(kChunk, std::max<uint64_t>(uint64_t(1) << 20,
                                                            (m / 8 + 31) & ~uint64_t(31)));
  const uint64_t chunk = std::min<uint64_t>(m, want_chunk);
  const size_t wbytes = align256((chunk + 31) / 32 * 4);
  size_t in_bytes = 0;
  if (!in_pinned)
    for (int k = 0; k < nin; ++k) in_bytes += align256(chunk * elt[k]);
  int rc = staging_reserve(st, pipe_slot_bytes(chunk, elt, nin));
  if (!rc) rc = host_reserve(st, in_bytes, 3 * wbytes);
  if (rc) return rc;
  PipeSlot slot[kSlots];
  for (int i = 0; i < kSlots; ++i) slot[i] = pipe_slot_view(st.buf[i], chunk, elt, nin);
  auto fail = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == kOk) rc = cuda_code(e);
    return rc != kOk;
  };
  auto want = [&](int e) {
    return (mask_words && mask_words[e]) || (mask_bytes && mask_bytes[e]);
  };
  for (int i = 0; i < kSlots && rc == kOk; ++i) fail(cudaMemsetAsync(slot[i].c, 0, 24, st.st[i]));
  const uint64_t nchunks = (m + chunk - 1) / chunk;
  auto finish = [&](uint64_t c) {  // chunk c's masks: pinned slot -> caller
    if (direct_out) {  // already in place; only the bounce slot's reuse waits
      if (!in_pinned) fail(cudaEventSynchronize(st.ev[c % kSlots]));
      return;
    }
    const int i = static_cast<int>(c % kSlots);
    if (fail(cudaEventSynchronize(st.ev[i]))) return;
    const uint64_t base = c * chunk, len = std::min<uint64_t>(chunk, m - base);
    for (int k = 0; k < ne; ++k) {
      const int e = eng[k];
      const uint32_t* hw = reinterpret_cast<const uint32_t*>(st.hout[i] + e * wbytes);
      if (mask_words && mask_words[e]) pool_memcpy(mask_words[e] + base / 32, hw, (len + 31) / 32 * 4);
      if (mask_bytes && mask_bytes[e]) pool_expand_bits(mask_bytes[e] + base, hw, len);
    }
  };
  uint64_t c = 0;
  for (; c < nchunks && rc == kOk; ++c) {
    const int i = static_cast<int>(c % kSlots);
    if (c >= kSlots && waits) finish(c - kSlots);
    if (rc) break;
    cudaStream_t s = st.st[i];
    const uint64_t base = c * chunk, len = std::min<uint64_t>(chunk, m - base);
    char* bounce = st.hin[i];
    for (int k = 0; k < nin && rc == kOk; ++k) {
      const void* src = static_cast<const char*>(hin[k]) + base * elt[k];
      if (!in_pinned) {
        pool_memcpy(bounce, src, len * elt[k]);
        src = bounce;
        bounce += align256(chunk * elt[k]);
      }
      fail(cudaMemcpyAsync(slot[i].in[k], src, len * elt[k], cudaMemcpyHostToDevice, s));
    }
    for (int k = 0; k < ne && rc == kOk; ++k) {
      const int e = eng[k];
      uint32_t* dw = want(e) ? slot[i].w[e] : nullptr;
      rc = launch(e, slot[i].in, len, dw, slot[i].c + e, s);
      if (!rc && dw)
        fail(cudaMemcpyAsync(direct_out ? static_cast<void*>(mask_words[e] + base / 32)
                                        : static_cast<void*>(st.hout[i] + e * wbytes),
                             dw, (len + 31) / 32 * 4, cudaMemcpyDeviceToHost, s));
    }
    if (rc == kOk) fail(cudaEventRecord(st.ev[i], s));
  }
  if (waits)
    for (uint64_t f = c > kSlots ? c - kSlots : 0; rc == kOk && f < c; ++f) finish(f);
  unsigned long long cnt[kSlots][3] = {};
  for (int i = 0; i < kSlots; ++i)
    if (rc == kOk) fail(cudaMemcpyAsync(cnt[i], slot[i].c, 24, cudaMemcpyDeviceToHost, st.st[i]));
  for (auto& s2 : st.st) fail(cudaStreamSynchronize(s2));
  if (rc == kOk && inside)
    for (int k = 0; k < ne; ++k) {
      inside[eng[k]] = 0;
      for (int i = 0; i < kSlots; ++i) inside[eng[k]] += cnt[i][eng[k]];
    }
  return rc;
}

}  // namespace

int vpipg_release_staging(int device) {
  if (device < 0 || device >= 64) return kInvalid;
  Staging& st = staging(device);
  std::lock_guard<std::mutex> lock(st.mu);
  if (!st.st[0] && !st.cap && !st.hcap_in) return kOk;
  DeviceGuard g(device);
  int rc = kOk;
  for (auto& s : st.st) {
    if (!s) continue;
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rc == kOk) rc = cuda_code(e);
    cudaStreamDestroy(s);
    s = nullptr;
  }
  for (auto& b : st.buf) {
    if (b) cudaFree(b);
    b = nullptr;
  }
  st.cap = 0;
  for (int i = 0; i < kSlots; ++i) {
    if (st.hin[i]) cudaFreeHost(st.hin[i]);
    if (st.hout[i]) cudaFreeHost(st.hout[i]);
    if (st.ev[i]) cudaEventDestroy(st.ev[i]);
    st.hin[i] = st.hout[i] = nullptr;
    st.ev[i] = nullptr;
  }
  st.hcap_in = st.hcap_out = 0;
  return rc;
}

int vpipg_test_host_multi(const vpipg_poly* p, uint32_t engines, int dtype, const void* xs,
                          const void* ys, uint64_t m, uint32_t* const* mask_words,
                          uint8_t* const* mask_bytes, uint64_t* inside) {
  if (!p || engines == 0 || (engines & ~7u)) return kInvalid;
  int eng[3], ne = 0;
  for (int e = 0; e < 3; ++e) {
    if (inside && (engines & (1u << e))) inside[e] = 0;
    if (engines & (1u << e)) eng[ne++] = e;
  }
  if (m == 0) return kOk;
  if (!xs || !ys) return kInvalid;
  DeviceGuard g(p->device);
  const size_t elt = dtype == VPIPG_F64 ? sizeof(double) : sizeof(float);
  bool want_bytes = false, pinned = host_pinned(xs) && host_pinned(ys);
  for (int k = 0; k < ne; ++k) {
    want_bytes |= mask_bytes && mask_bytes[eng[k]];
    if (mask_words) pinned = pinned && host_pinned(mask_words[eng[k]]);
    if (mask_bytes) pinned = pinned && host_pinned(mask_bytes[eng[k]]);
  }
  if (!pinned) {
    Staging& st = staging(p->device);
    std::lock_guard<std::mutex> lock(st.mu);
    const void* hin[2] = {xs, ys};
    const size_t el[2] = {elt, elt};
    return host_pipeline(st, hin, el, 2, m, eng, ne, mask_words, mask_bytes, inside,
                         [&](int e, void* const* din, uint64_t len, uint32_t* dw,
                             unsigned long long* dc, cudaStream_t s) {
                           TestArgs a{din[0], din[1], len, dw, nullptr, dc};
                           return dispatch(p, e, dtype, a, s);
                         });
  }
  // all-pinned buffers: DMA straight from / to the caller's memory in chunks,
  // kSlots in flight on their own streams: the points
  // cross PCIe once, every requested engine tests them, and the copy engines
  // stay busy in both directions
  // about 1/8 of the batch per chunk (1 Mi .. 16 Mi points) so copies in
  // both directions overlap the kernels even for mid-size batches
  const uint64_t chunk = std::min<uint64_t>(
      m, std::min<uint64_t>(kChunk, std::max<uint64_t>(uint64_t(1) << 20, (m / 8 + 31) & ~uint64_t(31))));
  Staging& st = staging(p->device);
  std::lock_guard<std::mutex> lock(st.mu);
  int rc = staging_reserve(st, slot_bytes(chunk, elt, want_bytes));
  if (rc) return rc;
  SlotView slot[kSlots];
  for (int i = 0; i < kSlots; ++i) slot[i] = slot_view(st.buf[i], chunk, elt, want_bytes);
  auto fail = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == kOk) rc = cuda_code(e);
    return rc != kOk;
  };
  for (int i = 0; i < kSlots && rc == kOk; ++i) fail(cudaMemsetAsync(slot[i].c, 0, 24, st.st[i]));
  const char* hx = static_cast<const char*>(xs);
  const char* hy = static_cast<const char*>(ys);
  for (uint64_t base = 0, c = 0; rc == kOk && base < m; base += chunk, ++c) {
    const int i = static_cast<int>(c % kSlots);
    cudaStream_t s = st.st[i];
    const uint64_t len = std::min<uint64_t>(chunk, m - base);
    if (fail(cudaMemcpyAsync(slot[i].x, hx + base * elt, len * elt, cudaMemcpyHostToDevice, s))) break;
    if (fail(cudaMemcpyAsync(slot[i].y, hy + base * elt, len * elt, cudaMemcpyHostToDevice, s))) break;
    for (int k = 0; k < ne && rc == kOk; ++k) {
      const int e = eng[k];
      uint32_t* dw = mask_words && mask_words[e] ? slot[i].w[e] : nullptr;
      uint8_t* db = mask_bytes && mask_bytes[e] ? slot[i].b[e] : nullptr;
      TestArgs a{slot[i].x, slot[i].y, len, dw, db, slot[i].c + e};
      rc = dispatch(p, e, dtype, a, s);
      if (rc) break;
      if (dw && fail(cudaMemcpyAsync(mask_words[e] + base / 32, dw, ((len + 31) / 32) * 4,
                                     cudaMemcpyDeviceToHost, s)))
        break;
      if (db && fail(cudaMemcpyAsync(mask_bytes[e] + base, db, len, cudaMemcpyDeviceToHost, s)))
        break;
    }
  }
  unsigned long long cnt[kSlots][3] = {};
  for (int i = 0; i < kSlots; ++i)
    if (rc == kOk) fail(cudaMemcpyAsync(cnt[i], slot[i].c, 24, cudaMemcpyDeviceToHost, st.st[i]));
  for (auto& s : st.st) fail(cudaStreamSynchronize(s));
  if (rc == kOk && inside)
    for (int k = 0; k < ne; ++k) {
      inside[eng[k]] = 0;
      for (int i = 0; i < kSlots; ++i) inside[eng[k]] += cnt[i][eng[k]];
    }
  return rc;
}

int vpipg_test_host(const vpipg_poly* p, int engine, int dtype, const void* xs, const void* ys,
                    uint64_t m, uint32_t* mask_words, uint8_t* mask_bytes, uint64_t* inside) {
  if (engine < 0 || engine > 2) return kInvalid;
  uint32_t* w[3] = {nullptr, nullptr, nullptr};
  uint8_t* b[3] = {nullptr, nullptr, nullptr};
  uint64_t cnt[3] = {0, 0, 0};
  w[engine] = mask_words;
  b[engine] = mask_bytes;
  const int rc = vpipg_test_host_multi(p, 1u << engine, dtype, xs, ys, m, w, b, cnt);
  if (inside) *inside = rc == kOk ? cnt[engine] : 0;
  return rc;
}


int vpipg_test_gather_host(const vpipg_db* db, uint32_t engines, const float* xs, const float* ys,
                           const uint32_t* ids, uint64_t m, uint32_t* const* mask_words,
                           uint8_t* const* mask_bytes, uint64_t* inside) {
  if (!db || engines == 0 || (engines & ~7u)) return kInvalid;
  int eng[3], ne = 0;
  for (int e = 0; e < 3; ++e) {
    if (!(engines & (1u << e))) continue;
    const uint32_t need = e == 0 ? kKindVoronoi : e == 1 ? kKindOffset : kKindCrossing;
    if (!(db->kinds & need)) return kInvalid;
    if (inside) inside[e] = 0;
    eng[ne++] = e;
  }
  if (m == 0) return kOk;
  if (!xs || !ys || !ids) return kInvalid;
  DeviceGuard g(db->device);
  Staging& st = staging(db->device);
  std::lock_guard<std::mutex> lock(st.mu);
  const void* hin[3] = {xs, ys, ids};
  const size_t el[3] = {sizeof(float), sizeof(float), sizeof(uint32_t)};
  return host_pipeline(st, hin, el, 3, m, eng, ne, mask_words, mask_bytes, inside,
                       [&](int e, void* const* din, uint64_t len, uint32_t* dw,
                           unsigned long long* dc, cudaStream_t s) {
                         GatherArgs a{static_cast<const float*>(din[0]),
                                      static_cast<const float*>(din[1]),
                                      static_cast<const uint32_t*>(din[2]), len, dw, nullptr, dc};
                         return cuda_code(launch_gather(db->t, e, a, s));
                       });
}

}  // extern "C"
