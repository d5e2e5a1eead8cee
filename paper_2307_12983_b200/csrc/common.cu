#include "common.h"

#include <cstdlib>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

namespace pqlg {

namespace {
thread_local std::string g_last_error;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || p == nullptr)
      throw Error(PQLG_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

int skip_step() {
  const char* e = std::getenv("PQLG_SKIP_STEP");
  return e ? std::atoi(e) : -1;
}

bool eager_updates() {
  static const bool on = [] {
    const char* e = std::getenv("PQLG_EAGER");
    return e && e[0] == '1';
  }();
  return on;
}

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                cudaGetErrorString(e), file, line, what);
  throw Error(PQLG_ECUDA, buf);
}

CUtensorMap make_tmap_2d(const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride,
                         uint32_t box_inner, uint32_t box_outer, Swz swz, bool tf32_type) {
  require((reinterpret_cast<uintptr_t>(base) & 15) == 0, "TMA base must be 16-byte aligned");
  require((row_stride * 4) % 16 == 0, "TMA row stride must be a multiple of 16 bytes");
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(
      &m, tf32_type ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      swz == Swz::k128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    std::snprintf(buf, sizeof(buf),
                  "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu stride=%llu box=%ux%u",
                  static_cast<int>(r), static_cast<unsigned long long>(inner),
                  static_cast<unsigned long long>(outer),
                  static_cast<unsigned long long>(row_stride), box_inner, box_outer);
    throw Error(PQLG_ECUDA, buf);
  }
  return m;
}

CUtensorMap make_tmap_3d(const void* base, uint64_t inner, uint64_t mid, uint64_t outer,
                         uint64_t stride_mid, uint64_t stride_outer, uint32_t box_inner,
                         uint32_t box_mid, Swz swz) {
  require((reinterpret_cast<uintptr_t>(base) & 15) == 0, "TMA base must be 16-byte aligned");
  require((stride_mid * 4) % 16 == 0 && (stride_outer * 4) % 16 == 0,
          "TMA strides must be multiples of 16 bytes");
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t dims[3] = {inner, mid, outer};
  cuuint64_t strides[2] = {stride_mid * 4, stride_outer * 4};
  cuuint32_t box[3] = {box_inner, box_mid, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE,
      swz == Swz::k128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(PQLG_ECUDA, "cuTensorMapEncodeTiled (3d) failed");
  return m;
}

std::atomic<uint64_t> g_launches{0};

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PQLG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace pqlg

extern "C" {
const char* pqlg_last_error(void) { return pqlg::g_last_error.c_str(); }
int pqlg_abi_version(void) { return 2; }  // 2: pqlg_config::precision
uint64_t pqlg_launch_count(void) { return pqlg::g_launches.load(); }
}

// ------------------------------------------------------------ launch profiler
namespace pqlg {

namespace {
struct ProfRec {
  cudaEvent_t a, b;
  const void* fn;
  std::string shape;
};
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_recs;
thread_local bool g_prof_skip = false;
// the instrumented capture of time_in_graph (this thread only)
thread_local std::vector<ProfRec>* t_graph_recs = nullptr;

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  return cs != cudaStreamCaptureStatusNone;
}
}  // namespace

bool profiling_active() {
  return t_graph_recs != nullptr || g_prof.load(std::memory_order_relaxed);
}

void profile_before(cudaStream_t st, const void* fn, const char* shape) {
  if (t_graph_recs) {  // instrumented capture: an event-record node in the graph
    ProfRec r{};
    r.fn = fn;
    if (shape) r.shape = shape;
    PQLG_CUDA(cudaEventCreate(&r.a));
    PQLG_CUDA(cudaEventCreate(&r.b));
    PQLG_CUDA(cudaEventRecordWithFlags(r.a, st, cudaEventRecordExternal));
    t_graph_recs->push_back(r);
    g_prof_skip = false;
    return;
  }
  g_prof_skip = capturing(st);
  if (g_prof_skip) return;
  ProfRec r{};
  r.fn = fn;
  PQLG_CUDA(cudaEventCreate(&r.a));
  PQLG_CUDA(cudaEventCreate(&r.b));
  PQLG_CUDA(cudaEventRecord(r.a, st));
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_recs.push_back(r);
}

void profile_after(cudaStream_t st) {
  if (t_graph_recs) {
    PQLG_CUDA(cudaEventRecordWithFlags(t_graph_recs->back().b, st, cudaEventRecordExternal));
    return;
  }
  if (g_prof_skip) return;
  cudaEvent_t b;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    b = g_prof_recs.back().b;
  }
  PQLG_CUDA(cudaEventRecord(b, st));
}

std::string time_in_graph(const std::function<void()>& enqueue, cudaStream_t st, int reps) {
  require(reps >= 1, "time_in_graph: reps must be >= 1");
  std::vector<ProfRec> recs;
  cudaEvent_t g0, g1;
  PQLG_CUDA(cudaEventCreate(&g0));
  PQLG_CUDA(cudaEventCreate(&g1));
  cudaGraph_t g = nullptr;
  const uint64_t before = g_launches.load();
  t_graph_recs = &recs;
  try {
    PQLG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    enqueue();
    PQLG_CUDA(cudaStreamEndCapture(st, &g));
  } catch (...) {
    t_graph_recs = nullptr;
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(st, &junk);
    if (junk) cudaGraphDestroy(junk);
    throw;
  }
  t_graph_recs = nullptr;
  const uint64_t per = g_launches.load() - before;
  g_launches.fetch_sub(per);  // captured, not launched
  cudaGraphExec_t ge;
  PQLG_CUDA(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  std::vector<double> acc(recs.size(), 0.0);
  double gacc = 0.0;
  for (int i = 0; i < reps + 2; ++i) {
    PQLG_CUDA(cudaEventRecord(g0, st));
    PQLG_CUDA(cudaGraphLaunch(ge, st));
    PQLG_CUDA(cudaEventRecord(g1, st));
    PQLG_CUDA(cudaStreamSynchronize(st));
    if (i < 2) continue;  // warm-up replays
    float ms = 0.0f;
    PQLG_CUDA(cudaEventElapsedTime(&ms, g0, g1));
    gacc += ms;
    for (size_t k = 0; k < recs.size(); ++k) {
      PQLG_CUDA(cudaEventElapsedTime(&ms, recs[k].a, recs[k].b));
      acc[k] += ms;
    }
  }
  count_launch(static_cast<uint64_t>(reps + 2) * per);
  std::string out;
  char buf[64];
  for (size_t k = 0; k < recs.size(); ++k) {
    const char* name = nullptr;
    if (cudaFuncGetName(&name, recs[k].fn) != cudaSuccess || !name) name = "?";
    std::snprintf(buf, sizeof(buf), "\t%.6f\t", acc[k] / reps);
    out += name;
    out += buf;
    out += recs[k].shape;
    out += '\n';
    cudaEventDestroy(recs[k].a);
    cudaEventDestroy(recs[k].b);
  }
  std::snprintf(buf, sizeof(buf), "__graph__\t%.6f\t\n", gacc / reps);
  out += buf;
  cudaGraphExecDestroy(ge);
  cudaEventDestroy(g0);
  cudaEventDestroy(g1);
  return out;
}
}  // namespace pqlg

extern "C" {

PQLG_API int pqlg_profile_begin(void) {
  return pqlg::guarded([] {
    std::lock_guard<std::mutex> lk(pqlg::g_prof_mu);
    for (auto& r : pqlg::g_prof_recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    pqlg::g_prof_recs.clear();
    pqlg::g_prof = true;
  });
}

// Writes "kernel-name\tmilliseconds\n" per profiled launch into out (NUL-
// terminated, truncated to cap bytes) and stops profiling.  Synchronizes.
PQLG_API int pqlg_profile_end(char* out, int cap) {
  return pqlg::guarded([&] {
    pqlg::g_prof = false;
    PQLG_CUDA(cudaDeviceSynchronize());
    std::string s;
    std::lock_guard<std::mutex> lk(pqlg::g_prof_mu);
    for (auto& r : pqlg::g_prof_recs) {
      float ms = 0.0f;
      PQLG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      const char* name = nullptr;
      if (cudaFuncGetName(&name, r.fn) != cudaSuccess || !name) name = "?";
      s += name;
      s += '\t';
      s += std::to_string(ms);
      s += '\n';
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    pqlg::g_prof_recs.clear();
    if (out && cap > 0) {
      const size_t n = std::min(static_cast<size_t>(cap - 1), s.size());
      std::memcpy(out, s.data(), n);
      out[n] = 0;
    }
  });
}

}  // extern "C"
