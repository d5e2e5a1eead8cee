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

// Orthogonal init (mlp.hpp:230-249): modified Gram-Schmidt on a
// normal_distribution<double> draw, in T = float, with -ffp-contract=off
// semantics (this TU is compiled without contraction for host code).
void init_orthogonal(const NetShape& net, std::vector<float>& flat, std::mt19937_64& rng,
                     float hidden_gain, float final_gain);

}  // namespace pqlg
