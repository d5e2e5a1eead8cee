// MetricsWriter (proj/include/pql/runtime/metrics.hpp:9-32,
// src/runtime/metrics.cpp:8-29): incremental CSV, header row then one
// flushed line per row, byte-identical to the reference's output.
#pragma once

#include <cstdio>
#include <mutex>
#include <string>

#include "pqlg.h"

namespace pqlg {

class MetricsWriter {
 public:
  static const char* header();
  explicit MetricsWriter(const std::string& path);
  ~MetricsWriter();
  MetricsWriter(const MetricsWriter&) = delete;
  MetricsWriter& operator=(const MetricsWriter&) = delete;
  void append(const pqlg_metrics_row& r);
  const std::string& path() const { return path_; }

 private:
  std::string path_;
  std::FILE* f_ = nullptr;
  std::mutex mu_;
};

// The loss EMAs of the metrics rows: the first sample seeds the average,
// then ema = f * ema + (1 - f) * x.
struct Ema {
  double f = 0.9, v = 0.0;
  bool seeded = false;
  void add(double x) {
    v = seeded ? f * v + (1.0 - f) * x : x;
    seeded = true;
  }
};

}  // namespace pqlg
