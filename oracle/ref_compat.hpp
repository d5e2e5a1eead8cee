// Pre-included (-include) when compiling the reference sources for
// oracle/_ref.  The reference does not compile as shipped:
// proj/include/pql/agents/policy.hpp:111 calls fa::forward(net, obs, nullptr)
// and template deduction fails on std::nullptr_t.  This adds the missing
// overload without touching the reference sources.
#pragma once

#include <cstddef>

#include "pql/funcapprox/mlp.hpp"

namespace pql::fa {
template <typename T>
Mat<T> forward(const Mlp<T>& net, const Mat<T>& in, std::nullptr_t) {
  return forward(net, in, static_cast<ForwardCache<T>*>(nullptr));
}
}  // namespace pql::fa
