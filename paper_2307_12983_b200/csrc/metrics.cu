// MetricsWriter (metrics.cpp:8-29) and its C ABI.
#include "metrics.h"

#include <memory>

#include "common.h"

namespace pqlg {

const char* MetricsWriter::header() {  // metrics.cpp:8-11
  return "wall_clock_s,env_steps,c_a,c_v,c_p,eval_return_mean,eval_return_stderr,"
         "critic_loss_ema,actor_loss_ema";
}

MetricsWriter::MetricsWriter(const std::string& path) : path_(path) {
  f_ = std::fopen(path.c_str(), "w");  // std::ios::trunc
  if (!f_) throw Error(PQLG_EINVAL, "metrics: cannot open " + path);
  std::fputs(header(), f_);
  std::fputc('\n', f_);
  std::fflush(f_);
}

MetricsWriter::~MetricsWriter() {
  if (f_) std::fclose(f_);
}

void MetricsWriter::append(const pqlg_metrics_row& r) {  // metrics.cpp:19-27
  char buf[320];
  std::snprintf(buf, sizeof(buf), "%.3f,%lld,%lld,%lld,%lld,%.6g,%.6g,%.6g,%.6g",
                r.wall_clock_s, static_cast<long long>(r.env_steps),
                static_cast<long long>(r.c_a), static_cast<long long>(r.c_v),
                static_cast<long long>(r.c_p), r.eval_return_mean, r.eval_return_stderr,
                r.critic_loss_ema, r.actor_loss_ema);
  std::lock_guard<std::mutex> lk(mu_);
  std::fputs(buf, f_);
  std::fputc('\n', f_);
  std::fflush(f_);  // one flushed line per row: a crash loses at most the row in flight
}

}  // namespace pqlg

struct pqlg_metrics_s {
  std::unique_ptr<pqlg::MetricsWriter> w;
};

using namespace pqlg;

extern "C" {

const char* pqlg_metrics_header(void) { return MetricsWriter::header(); }

int pqlg_metrics_open(const char* path, pqlg_metrics* out) {
  return guarded([&] {
    require(path && out, "metrics_open: null argument");
    auto h = std::make_unique<pqlg_metrics_s>();
    h->w = std::make_unique<MetricsWriter>(path);
    *out = h.release();
  });
}

int pqlg_metrics_append(pqlg_metrics h, const pqlg_metrics_row* row) {
  return guarded([&] {
    require(h && row, "metrics_append: null argument");
    h->w->append(*row);
  });
}

int pqlg_metrics_close(pqlg_metrics h) {
  return guarded([&] { delete h; });
}

void pqlg_metrics_config_default(pqlg_metrics_config* m) {
  *m = pqlg_metrics_config{};
  m->path = nullptr;
  m->interval_s = 5.0;
  m->every_actor_steps = 1000;
  m->eval_episodes = 64;
  m->eval_seed = 12345;
  m->ema = 0.9;
}

}  // extern "C"
