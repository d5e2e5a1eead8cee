#include "pdl.cuh"
#include "net.h"

namespace pqlg {

namespace {
__global__ void pad_rows_kernel(const float* src, float* dst, int rows, int cols, int ld) {
  pdl::entry();
  const int64_t n = static_cast<int64_t>(rows) * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    dst[r * ld + c] = src[i];
  }
}
}  // namespace

void launch_pad_rows(const float* src, float* dst, int rows, int cols, int ld, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(rows) * cols;
  const int blocks = static_cast<int>(std::min<int64_t>(592, (n + 255) / 256));
  launch(pad_rows_kernel, dim3(blocks), dim3(256), 0, st, src, dst, rows, cols, ld);
}

namespace {
struct PadMulti {
  const float* src[4];
  float* dst[4];
  int rows, cols, ld;
};
__global__ void pad_rows_multi_kernel(const __grid_constant__ PadMulti a) {
  pdl::entry();
  const int k = blockIdx.y;
  const int64_t n = static_cast<int64_t>(a.rows) * a.cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / a.cols, c = i % a.cols;
    a.dst[k][r * a.ld + c] = a.src[k][i];
  }
}
}  // namespace

void refresh_mirrors(const WeightMirror* m, int n, cudaStream_t st) {
  if (n <= 0 || !m[0].needed()) return;
  require(n <= 4, "refresh_mirrors: at most 4");
  PadMulti a{};
  for (int k = 0; k < n; ++k) {
    require(m[k].in == m[0].in && m[k].out == m[0].out, "refresh_mirrors: shapes differ");
    a.src[k] = m[k].src;
    a.dst[k] = m[k].buf.p;
  }
  a.rows = m[0].in;
  a.cols = m[0].out;
  a.ld = m[0].ld;
  const int64_t total = static_cast<int64_t>(a.rows) * a.cols;
  const int blocks = static_cast<int>(std::min<int64_t>(148, (total + 255) / 256));
  launch(pad_rows_multi_kernel, dim3(blocks, n), dim3(256), 0, st, a);
}

namespace {
// detail::orthogonalize (mlp.hpp:209-225), T = float.
void orthogonalize(std::vector<float>& a, size_t rows, size_t cols) {
  for (size_t c = 0; c < cols; ++c) {
    for (size_t p = 0; p < c; ++p) {
      float dot = 0.0f;
      for (size_t r = 0; r < rows; ++r) dot += a[r * cols + c] * a[r * cols + p];
      for (size_t r = 0; r < rows; ++r) a[r * cols + c] -= dot * a[r * cols + p];
    }
    float norm = 0.0f;
    for (size_t r = 0; r < rows; ++r) norm += a[r * cols + c] * a[r * cols + c];
    norm = std::sqrt(norm);
    if (norm < 1e-12f) norm = 1.0f;
    for (size_t r = 0; r < rows; ++r) a[r * cols + c] /= norm;
  }
}
}  // namespace

void init_orthogonal(const NetShape& net, std::vector<float>& flat, std::mt19937_64& rng,
                     float hidden_gain, float final_gain) {
  flat.assign(net.params, 0.0f);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int l = 0; l < net.layers(); ++l) {
    const size_t in = net.sizes[l], out = net.sizes[l + 1];
    const size_t big = std::max(in, out), small = std::min(in, out);
    std::vector<float> m(big * small);
    for (auto& x : m) x = static_cast<float>(gauss(rng));
    orthogonalize(m, big, small);
    const float gain = (l + 1 == net.layers()) ? final_gain : hidden_gain;
    float* w = flat.data() + net.w_off[l];
    for (size_t i = 0; i < in; ++i)
      for (size_t o = 0; o < out; ++o) {
        const float v = (in >= out) ? m[i * small + o] : m[o * small + i];
        w[i * out + o] = gain * v;
      }
    float* b = flat.data() + net.b_off[l];
    for (size_t o = 0; o < out; ++o) b[o] = 0.0f;
  }
}

}  // namespace pqlg
