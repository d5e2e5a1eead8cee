// Traced copy of the forward-layer GEMM (tools only): per-CTA phase
// timestamps to split a launch into prologue / pipeline fill / mainloop /
// epilogue.  Build: see tools/gemm_trace.py.
#define PQLG_GEMM_TRACE 1
#include "../paper_2307_12983_b200/csrc/epilogues.cuh"
#include "../paper_2307_12983_b200/csrc/gemm_host.cuh"

using namespace pqlg;

// kind 0: hidden layer (BN 256, Hidden epilogue); 1: policy head (BN 32,
// PolicyHead: bias + tanh squash, no noise) with N <= 32.
extern "C" __attribute__((visibility("default"))) int trace_gemm(
    const float* A, const float* B, float* D, const float* bias, int M, int N, int K, int groups,
    unsigned long long* trace, int iters, int store, int kind, void* stream) {
  return guarded([&] {
    auto st = static_cast<cudaStream_t>(stream);
    PQLG_CUDA(cudaMemcpyToSymbol(gemm::g_trace, &trace, sizeof(trace)));
    gemm::Operands ops;
    const gemm::Problem p = gemm::make_problem(M, N, K, 1);
    if (kind == 0) {
      ops.a[0] = ops.a[1] = ops.a[2] = ops.a[3] = gemm::map_a(A, M, K, K, false, true);
      ops.b[0] = ops.b[1] = ops.b[2] = ops.b[3] = gemm::map_b(B, N, K, N, true, 256, true);
      ops.d[0] = ops.d[1] = ops.d[2] = ops.d[3] = make_store_map(D, M, N, N);
      epi::Hidden e{};
      e.bias[0] = e.bias[1] = e.bias[2] = e.bias[3] = bias;
      e.bn = 256;
      e.M = M;
      e.N = N;
      e.store = store ? 0xF : 0;
      for (int i = 0; i < iters; ++i) gemm::launch<256, false, true>(ops, p, groups, e, st);
    } else {
      if (kind == 2) {
        // in situ: the preceding hidden layer writes the head's input (A)
        // right before the head, as in the update / actor step
        PQLG_CUDA(cudaMemcpyToSymbol(gemm::g_trace, &trace, sizeof(trace)));
        unsigned long long* none = nullptr;
        PQLG_CUDA(cudaMemcpyToSymbol(gemm::g_trace, &none, sizeof(none)));
        gemm::Operands h;
        for (int g = 0; g < 4; ++g) {
          h.a[g] = gemm::map_a(D, M, K, K, false, true);  // D doubles as the hidden input
          h.b[g] = gemm::map_b(B, K, K, K, true, 256, true);
          h.d[g] = make_store_map(const_cast<float*>(A), M, K, K);
        }
        epi::Hidden e{};
        for (int g = 0; g < 4; ++g) e.bias[g] = bias;
        e.bn = 256;
        e.M = M;
        e.N = K;
        e.store = 1;
        gemm::launch<256, false, true>(h, gemm::make_problem(M, K, K, 1), 1, e, st);
        PQLG_CUDA(cudaMemcpyToSymbol(gemm::g_trace, &trace, sizeof(trace)));
      }
      ops.a[0] = ops.a[1] = ops.a[2] = ops.a[3] = gemm::map_a(A, M, K, K, false, true);
      ops.b[0] = ops.b[1] = gemm::map_b(B, N, K, N, true, 32, true);
      epi::PolicyHead e{};
      e.bias = bias;
      e.act = D;
      e.ld_act = N;
      e.M = M;
      e.A = N;
      e.mid = 0.0f;
      e.half = 1.0f;
      for (int i = 0; i < iters; ++i) gemm::launch<32, false, true>(ops, p, groups, e, st);
    }
  });
}
