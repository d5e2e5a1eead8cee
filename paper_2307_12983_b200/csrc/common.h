// Host-side plumbing shared by every translation unit of libpqlg: status
// codes, the thread-local last-error string, CUDA error checking and TMA
// tensor-map construction.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <algorithm>
#include <cstring>
#include <functional>
#include <string>
#include <utility>

#include "../../include/pqlg.h"

namespace pqlg {

// Exceptions carry the C status they map to at the ABI boundary.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define PQLG_CUDA(expr)                                                   \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) ::pqlg::throw_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)

#define PQLG_CHECK_LAUNCH() PQLG_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(PQLG_EINVAL, msg);
}

void set_last_error(const std::string& msg);

// Kernel launches issued by this library (reported through pqlg_launch_count).
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Every library kernel is launched through launch(): with the programmatic
// stream-serialisation attribute (PDL, see pdl.cuh) unless PQLG_PDL=0.
bool pdl_enabled();

// Per-launch device timing (pqlg_profile_begin/end): when active, launch()
// brackets every kernel issued outside stream capture with a pair of events.
// During an instrumented capture (time_in_graph) the same hooks record
// event-record nodes into the graph instead, so kernels are timed as they run
// inside the replayed graph.  `shape` describes GEMM launches (groups, M, N, K).
bool profiling_active();
void profile_before(cudaStream_t st, const void* fn, const char* shape = nullptr);
void profile_after(cudaStream_t st);

// Captures enqueue() on `st` into a graph with an event-record node before
// and after every library kernel, replays it `reps` times (after 2 warm-up
// replays) and returns "kernel\tavg_ms\tshape\n" per launch in launch order,
// followed by "__graph__\tavg_ms\t\n" (the whole instrumented replay).
// The event nodes break programmatic-dependent-launch overlap between
// neighbours, so these are per-kernel durations without PDL prologue overlap.
// NUL-terminated copy into a caller buffer of `cap` bytes (truncating).
inline void copy_cstr(const std::string& s, char* out, int cap) {
  const size_t n = std::min(static_cast<size_t>(cap - 1), s.size());
  std::memcpy(out, s.data(), n);
  out[n] = 0;
}

std::string time_in_graph(const std::function<void()>& enqueue, cudaStream_t st, int reps);

template <class... KArgs, class... Args>
void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
            Args&&... args) {
  const bool prof = profiling_active();
  if (prof) profile_before(st, reinterpret_cast<const void*>(kernel));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PQLG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  count_launch();
  if (prof) profile_after(st);
}

// Profiling aid: PQLG_SKIP_STEP=i drops step i of an update's launch list
// when it is (re)built, so graph replays measure each step's marginal cost
// in situ (results are then meaningless; tools/skip_probe.py).
int skip_step();
// Profiling aid: PQLG_EAGER=1 makes update() launch its kernels one by one
// (the launch profiler brackets each) instead of replaying the update graph.
bool eager_updates();

// Wraps an ABI entry point: converts exceptions to status codes.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return PQLG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PQLG_EINVAL;
  }
}

// Owning device allocation (cudaMalloc; zero-initialised before alloc()
// returns: cudaMemset is queued on the legacy stream, which does not order
// with the library's non-blocking streams, so without the wait a kernel
// launched right after construction could run before the zeroing lands and
// have its writes (counters, normalizer state) zeroed after it).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) {
      PQLG_CUDA(cudaMalloc(&p, count * sizeof(T)));
      PQLG_CUDA(cudaMemset(p, 0, count * sizeof(T)));
      PQLG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
  T* get() const { return p; }
};

// Synchronous copy for construction-time setup: cudaMemcpy can return before
// an H2D (pageable) or D2D copy has landed, on the legacy stream, which does
// not order with the library's non-blocking streams; wait for it.
inline void copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  PQLG_CUDA(cudaMemcpy(dst, src, bytes, kind));
  PQLG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
}

// Owning pinned host allocation (cudaMallocHost): truly asynchronous copies.
template <class T>
struct PinnedBuf {
  T* p = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void alloc(size_t count) {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = count;
    if (count) PQLG_CUDA(cudaMallocHost(&p, count * sizeof(T)));
  }
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ----------------------------------------------------------------- TMA maps
enum class Swz { k128, k128a32 };

// 2-D fp32 tensor map: `inner` contiguous elements per row, `outer` rows at
// `row_stride` elements; box = box_inner x box_outer elements.
CUtensorMap make_tmap_2d(const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride,
                         uint32_t box_inner, uint32_t box_outer, Swz swz, bool tf32_type = false);

// 3-D fp32 tensor map {inner, mid, outer}; strides in elements.
CUtensorMap make_tmap_3d(const void* base, uint64_t inner, uint64_t mid, uint64_t outer,
                         uint64_t stride_mid, uint64_t stride_outer, uint32_t box_inner,
                         uint32_t box_mid, Swz swz);

// Output map of a GEMM epilogue: rows x cols fp32, box 32 x 32, 128B swizzle.
inline CUtensorMap make_store_map(const void* base, uint64_t rows, uint64_t cols, uint64_t ld) {
  return make_tmap_2d(base, cols, rows, ld, 32, 32, Swz::k128, false);
}

}  // namespace pqlg
