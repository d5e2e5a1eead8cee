"""Builds the reference-side B200 binding from the reference's
own files, at build time, into oracle/_ref/b200/ (git-ignored; the reference
sources are never copied into the repository).

What a maintainer adds to /root/reference/proj under `PQL_B200`:
  include/pql/runtime/learners.hpp   a handful of #ifdef lines (below):
      - include pqlg.hpp and a PQL_B200_MUTABLE helper
      - an opaque `std::shared_ptr<B200> b200_` member in each core
      - out-of-line accessors whose host state the device now owns
        (CriticLearnerCore::critics / buffer_size, PolicyLearnerCore::
        ingest / policy / buffer_size), their members made mutable
  src/runtime/learners.cpp           the three cores' definitions
      (learners.cpp:58-274) wrapped in #ifndef PQL_B200, with
      #include "b200_cores.inc" (this directory) in the #else branch
Each edit below asserts its anchor, so a change in the reference fails the
build loudly instead of producing a silently different binding.

    python oracle/b200_binding/make_binding.py REF_PROJ OUT_DIR
"""
from __future__ import annotations

import sys
from pathlib import Path


def edit(text: str, old: str, new: str, count: int = 1) -> str:
    n = text.count(old)
    if n != count:
        raise SystemExit(f"make_binding: anchor found {n} times (want {count}):\n{old}")
    return text.replace(old, new)


def patch_header(h: str) -> str:
    h = edit(h, '#include "pql/vecenv/vecenv.hpp"\n',
             '#include "pql/vecenv/vecenv.hpp"\n'
             '\n#ifdef PQL_B200\n#include <cstdlib>\n#include <cstring>\n'
             '#include "pqlg.hpp"  // B200 path: libpqlg.so (include/pqlg.h)\n'
             '#define PQL_B200_MUTABLE mutable\n#else\n#define PQL_B200_MUTABLE\n#endif\n')
    b200_member = '#ifdef PQL_B200\n  struct B200;  // the device core (b200_cores.inc)\n' \
                  '  std::shared_ptr<B200> b200_;\n#endif\n};'
    h = edit(h, '  std::vector<env::SplitMixEngine> noise_rng_;\n};',
             '  std::vector<env::SplitMixEngine> noise_rng_;\n' + b200_member)
    h = edit(h, '  std::mt19937_64 sample_rng_, eps_rng_;\n};',
             '  std::mt19937_64 sample_rng_, eps_rng_;\n' + b200_member, count=2)
    crit = ('  const agents::CriticPair<float>& critics() const { return critics_; }\n'
            '  std::size_t buffer_size() const { return buffer_.size(); }\n')
    h = edit(h, crit, '#ifdef PQL_B200\n'
                      '  const agents::CriticPair<float>& critics() const;  // synced from the device\n'
                      '  std::size_t buffer_size() const;\n#else\n' + crit + '#endif\n')
    h = edit(h, '  agents::CriticPair<float> critics_;\n',
             '  PQL_B200_MUTABLE agents::CriticPair<float> critics_;\n')
    h = edit(h, '  agents::CriticPair<float> critics_;  // online replicas',
             '  PQL_B200_MUTABLE agents::CriticPair<float> critics_;  // online replicas')
    ing = '  void ingest(const MatF& states) { state_buf_.insert(states); }\n'
    h = edit(h, ing, '#ifdef PQL_B200\n  void ingest(const MatF& states);\n#else\n' + ing +
             '#endif\n')
    pol = ('  const PolicyHandle& policy() const { return policy_; }\n'
           '  std::size_t buffer_size() const { return state_buf_.size(); }\n')
    h = edit(h, pol, '#ifdef PQL_B200\n'
                     '  const PolicyHandle& policy() const;  // synced from the device\n'
                     '  std::size_t buffer_size() const;\n#else\n' + pol + '#endif\n')
    # PolicyLearnerCore's policy_ (the second PolicyHandle policy_ member)
    i = h.index('class PolicyLearnerCore')
    tail = edit(h[i:], '  PolicyHandle policy_;\n', '  PQL_B200_MUTABLE PolicyHandle policy_;\n')
    return h[:i] + tail


def patch_source(c: str) -> str:
    sep = '// ' + '-' * 75 + '\n'
    start = sep + '// ActorCore\n'
    if c.count(start) != 1:
        raise SystemExit("make_binding: ActorCore section header not found")
    c = c.replace(start, '#ifndef PQL_B200\n' + start)
    end = ('PolicySnapshot PolicyLearnerCore::make_snapshot(std::int64_t version) const {\n'
           '  return policy_.snapshot(version, norm_);\n}\n')
    c = edit(c, end, end + '\n#else  // PQL_B200: the cores bind to the device path\n'
                           '#include "b200_cores.inc"\n#endif  // PQL_B200\n')
    return c


def main():
    ref, out = Path(sys.argv[1]), Path(sys.argv[2])
    (out / "include" / "pql" / "runtime").mkdir(parents=True, exist_ok=True)
    h = (ref / "include" / "pql" / "runtime" / "learners.hpp").read_text()
    c = (ref / "src" / "runtime" / "learners.cpp").read_text()
    (out / "include" / "pql" / "runtime" / "learners.hpp").write_text(patch_header(h))
    (out / "learners.cpp").write_text(patch_source(c))


if __name__ == "__main__":
    main()
