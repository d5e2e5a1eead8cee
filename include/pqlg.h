/*
 * pqlg.h -- C ABI of the B200-native PQL learner/actor hot path (libpqlg.so).
 *
 * Drop-in boundary for the reference's runtime cores and replay objects
 * (reference paths are relative to /root/reference):
 *   ReplayBuffer / StateBuffer     proj/include/pql/replay/replay_buffer.hpp:17-119
 *   NStepAssembler / NStepBatch    proj/include/pql/replay/nstep.hpp:15-126
 *   ActorCore                      proj/include/pql/runtime/learners.hpp:52-73
 *   CriticLearnerCore              proj/include/pql/runtime/learners.hpp:77-106
 *   PolicyLearnerCore              proj/include/pql/runtime/learners.hpp:110-139
 *   kernels::* operator API        proj/include/pql/kernels/kernels.hpp:17-83
 *
 * Conventions
 *   - Every entry point returns an int status (PQLG_*); pqlg_last_error()
 *     returns the thread-local message of the last failure.
 *   - Pointers named *_dev are device pointers; *_host are host pointers.
 *   - Handles are owned by one host thread and run on one CUDA stream; all
 *     device work is asynchronous on that stream unless stated otherwise.
 *   - The library has no CPU fallback: without a CUDA device every compute
 *     entry point fails with PQLG_ECUDA.
 */
#ifndef PQLG_H_
#define PQLG_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PQLG_API __attribute__((visibility("default")))
#else
#define PQLG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum {
  PQLG_OK = 0,
  PQLG_NOT_READY = 1,   /* empty std::optional / "before warm-up" runtime_error */
  PQLG_EINVAL = -1,     /* std::invalid_argument (shape / config)               */
  PQLG_ENONFINITE = -2, /* std::runtime_error for non-finite values             */
  PQLG_ECUDA = -3,
  PQLG_ENCCL = -4
};

PQLG_API const char* pqlg_last_error(void);
PQLG_API int pqlg_abi_version(void);
/* Number of kernels this library launched since load (evidence counter). */
PQLG_API uint64_t pqlg_launch_count(void);

/* ------------------------------------------------- operator-level test hooks
 * Device-pointer restatements of pql::kernels (kernels.hpp:25-60); there is
 * no backend dispatch -- these run the sm_100a kernels the learners use.
 */

/* D[M x N] = A x B (+ bias, ReLU) on tcgen05 tensor cores (tf32 inputs,
 * fp32 accumulate).  a_mn = 0: A is [M x K] row-major (K contiguous, stride
 * lda); a_mn = 1: A is stored transposed as [K x M] (stride lda).
 * b_mn = 0: B stored as [N x K] (stride ldb); b_mn = 1: B is [K x N].
 * splits > 1 splits K across CTAs with a fixed-order reduction.
 * round_mode: 0 = operands fed as fp32 bit patterns (hardware tf32 reads),
 *             1 = TMA tensor maps typed TFLOAT32. */
PQLG_API int pqlg_k_gemm_tf32(const float* A_dev, const float* B_dev, float* D_dev, const float* bias_dev,
                     int M, int N, int K, int a_mn, int b_mn, int lda, int ldb, int ldd, int relu,
                     int splits, int round_mode, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PQLG_H_ */
