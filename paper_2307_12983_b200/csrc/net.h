// Flat-parameter MLPs on device (fa::Mlp layout, mlp.hpp:68-91: per layer
// W [in x out] row-major then b) and the host-side orthogonal init that
// reproduces fa::init_orthogonal (mlp.hpp:230-249) bit for bit.
#pragma once

#include <cmath>
#include <random>
#include <vector>

#include "common.h"

namespace pqlg {

struct NetShape {
  std::vector<int> sizes;  // in, hidden..., out
  std::vector<int64_t> w_off, b_off;
  int64_t params = 0;

  static NetShape make(const std::vector<int>& s) {
    NetShape n;
    n.sizes = s;
    int64_t t = 0;
    for (size_t l = 0; l + 1 < s.size(); ++l) {
      n.w_off.push_back(t);
      t += static_cast<int64_t>(s[l]) * s[l + 1];
      n.b_off.push_back(t);
      t += s[l + 1];
    }
    n.params = t;
    return n;
  }
  int layers() const { return static_cast<int>(sizes.size()) - 1; }
  int in() const { return sizes.front(); }
  int out() const { return sizes.back(); }
};

// dst[r * ld + c] = src[r * cols + c] (c < cols); padding columns stay zero.
void launch_pad_rows(const float* src, float* dst, int rows, int cols, int ld, cudaStream_t st);

// TMA needs 16-byte row strides: a weight matrix W [in x out] whose `out` is
// not a multiple of 4 (policy heads with act_dim 1/2/3, the 51-atom C51
// head) is read by the GEMMs from a padded mirror refreshed after every
// parameter change.
struct WeightMirror {
  const float* src = nullptr;
  int in = 0, out = 0, ld = 0;
  DevBuf<float> buf;
  void init(const float* w, int rows, int cols) {
    src = w;
    in = rows;
    out = cols;
    ld = static_cast<int>(round_up(cols, 4));
    if (ld != cols) buf.alloc(static_cast<size_t>(rows) * ld);
  }
  bool needed() const { return buf.p != nullptr; }
  const float* ptr() const { return needed() ? buf.p : src; }
  int64_t stride() const { return needed() ? ld : out; }
  void refresh(cudaStream_t st) const {
    if (needed()) launch_pad_rows(src, buf.p, in, out, ld, st);
  }
};

// Refreshes up to 4 mirrors of the same shape in one launch.
void refresh_mirrors(const WeightMirror* m, int n, cudaStream_t st);

// CategoricalHead::create (c51.hpp:21-34): z_j = float(vmin + dz*j) in fp64,
// the end points exact.
inline std::vector<float> c51_atoms(int L, float vmin, float vmax) {
  std::vector<float> z(L);
  const double dz = (static_cast<double>(vmax) - vmin) / static_cast<double>(L - 1);
  for (int j = 0; j < L; ++j) z[j] = static_cast<float>(static_cast<double>(vmin) + dz * j);
  z.front() = vmin;
  z.back() = vmax;
  return z;
}

// Orthogonal init (mlp.hpp:230-249): modified Gram-Schmidt on a
// normal_distribution<double> draw, in T = float, with -ffp-contract=off
// semantics (this TU is compiled without contraction for host code).
void init_orthogonal(const NetShape& net, std::vector<float>& flat, std::mt19937_64& rng,
                     float hidden_gain, float final_gain);

}  // namespace pqlg
