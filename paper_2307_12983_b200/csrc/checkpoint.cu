// Checkpoints in the reference's on-disk format (fa::save_checkpoint /
// load_checkpoint, proj/src/funcapprox/checkpoint.cpp:35-91, SURVEY §8(f)
// rank 2): "PQLCKPT\x01", u32 net count, per net (u32 name length, name,
// u32 layer-size count, u32 sizes, u8 activation per layer, f32 params in the
// flat Mlp layout), then u32 dim, i64 count, f64 mean[dim], f64 m2[dim] --
// all little-endian.  Host code: the learners stage parameters through host
// copies (the files are byte-identical to the reference's, tests/test_checkpoint_cpu.py).
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "actor.h"
#include "learner.h"

namespace pqlg::ckpt {
namespace {

constexpr char kMagic[8] = {'P', 'Q', 'L', 'C', 'K', 'P', 'T', '\x01'};

struct Net {
  std::string name;
  std::vector<uint32_t> sizes;
  std::vector<uint8_t> acts;
  std::vector<float> flat;
};
struct File {
  std::vector<Net> nets;
  int64_t count = 0;
  std::vector<double> mean, m2;
};

template <class T>
void put(std::ofstream& f, T v) {
  f.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <class T>
T get(std::ifstream& f) {
  T v;
  f.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!f) throw Error(PQLG_EINVAL, "checkpoint: truncated file");
  return v;
}

void write(const std::string& path, const File& c) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw Error(PQLG_EINVAL, "checkpoint: cannot open " + path);
  f.write(kMagic, sizeof(kMagic));
  put<uint32_t>(f, static_cast<uint32_t>(c.nets.size()));
  for (const Net& n : c.nets) {
    put<uint32_t>(f, static_cast<uint32_t>(n.name.size()));
    f.write(n.name.data(), static_cast<std::streamsize>(n.name.size()));
    put<uint32_t>(f, static_cast<uint32_t>(n.sizes.size()));
    for (uint32_t s : n.sizes) put<uint32_t>(f, s);
    for (uint8_t a : n.acts) put<uint8_t>(f, a);
    f.write(reinterpret_cast<const char*>(n.flat.data()),
            static_cast<std::streamsize>(n.flat.size() * sizeof(float)));
  }
  put<uint32_t>(f, static_cast<uint32_t>(c.mean.size()));
  put<int64_t>(f, c.count);
  f.write(reinterpret_cast<const char*>(c.mean.data()),
          static_cast<std::streamsize>(c.mean.size() * sizeof(double)));
  f.write(reinterpret_cast<const char*>(c.m2.data()),
          static_cast<std::streamsize>(c.m2.size() * sizeof(double)));
  if (!f) throw Error(PQLG_EINVAL, "checkpoint: write failed for " + path);
}

int64_t param_count(const std::vector<uint32_t>& sizes) {
  int64_t t = 0;
  for (size_t l = 0; l + 1 < sizes.size(); ++l)
    t += static_cast<int64_t>(sizes[l]) * sizes[l + 1] + sizes[l + 1];
  return t;
}

File read(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error(PQLG_EINVAL, "checkpoint: cannot open " + path);
  char magic[8];
  f.read(magic, sizeof(magic));
  if (!f || std::memcmp(magic, kMagic, sizeof(kMagic)) != 0)
    throw Error(PQLG_EINVAL, "checkpoint: bad magic/version in " + path);
  File c;
  const uint32_t n_nets = get<uint32_t>(f);
  for (uint32_t k = 0; k < n_nets; ++k) {
    Net n;
    n.name.resize(get<uint32_t>(f));
    f.read(n.name.data(), static_cast<std::streamsize>(n.name.size()));
    const uint32_t ns = get<uint32_t>(f);
    if (ns < 2) throw Error(PQLG_EINVAL, "checkpoint: bad layer count");
    n.sizes.resize(ns);
    for (auto& s : n.sizes) s = get<uint32_t>(f);
    n.acts.resize(ns - 1);
    for (auto& a : n.acts) a = get<uint8_t>(f);
    n.flat.resize(param_count(n.sizes));
    f.read(reinterpret_cast<char*>(n.flat.data()),
           static_cast<std::streamsize>(n.flat.size() * sizeof(float)));
    if (!f) throw Error(PQLG_EINVAL, "checkpoint: truncated parameters");
    c.nets.push_back(std::move(n));
  }
  const uint32_t dim = get<uint32_t>(f);
  c.count = get<int64_t>(f);
  c.mean.resize(dim);
  c.m2.resize(dim);
  f.read(reinterpret_cast<char*>(c.mean.data()), static_cast<std::streamsize>(dim * 8));
  f.read(reinterpret_cast<char*>(c.m2.data()), static_cast<std::streamsize>(dim * 8));
  if (!f) throw Error(PQLG_EINVAL, "checkpoint: truncated normalizer");
  return c;
}

// the learners' nets: ReLU hidden layers, identity output (learners.cpp:20-30)
Net make_net(const std::string& name, const NetShape& shape, std::vector<float> flat) {
  Net n;
  n.name = name;
  for (int s : shape.sizes) n.sizes.push_back(static_cast<uint32_t>(s));
  n.acts.assign(shape.sizes.size() - 1, 1);
  n.acts.back() = 0;
  n.flat = std::move(flat);
  return n;
}

const Net& find(const File& c, const std::string& name, const NetShape& shape) {
  for (const Net& n : c.nets)
    if (n.name == name) {
      std::vector<uint32_t> want(shape.sizes.begin(), shape.sizes.end());
      if (n.sizes != want) throw Error(PQLG_EINVAL, "checkpoint: net '" + name + "' shape mismatch");
      return n;
    }
  throw Error(PQLG_EINVAL, "checkpoint: no net named '" + name + "'");
}

void set_norm(File& c, int64_t count, const std::vector<double>& mean, const std::vector<double>& m2,
              int D) {
  c.count = count;
  c.mean = mean.empty() ? std::vector<double>(D, 0.0) : mean;
  c.m2 = m2.empty() ? std::vector<double>(D, 0.0) : m2;
}

}  // namespace
}  // namespace pqlg::ckpt

using namespace pqlg;
using namespace pqlg::ckpt;

extern "C" {

int pqlg_checkpoint_write(const char* path, int n_nets, const char* const* names,
                          const int32_t* n_layers, const int32_t* const* sizes,
                          const float* const* flats, int64_t count, const double* mean,
                          const double* m2, int dim) {
  return guarded([&] {
    require(path && (n_nets == 0 || (names && n_layers && sizes && flats)),
            "checkpoint_write: null argument");
    File c;
    for (int k = 0; k < n_nets; ++k) {
      require(n_layers[k] >= 1, "checkpoint_write: nets need >= 1 layer");
      std::vector<int> s(sizes[k], sizes[k] + n_layers[k] + 1);
      const NetShape shape = NetShape::make(s);
      c.nets.push_back(make_net(names[k], shape,
                                std::vector<float>(flats[k], flats[k] + shape.params)));
    }
    c.count = count;
    c.mean.assign(mean, mean + dim);
    c.m2.assign(m2, m2 + dim);
    write(path, c);
  });
}

int pqlg_checkpoint_read(const char* path, int* n_nets, int64_t* n_params, float* flat_out,
                         int64_t* count, double* mean, double* m2, int* dim) {
  return guarded([&] {
    require(path && n_nets && n_params && count && dim, "checkpoint_read: null argument");
    const File c = read(path);
    int64_t total = 0;
    for (const Net& n : c.nets) {
      if (flat_out) std::memcpy(flat_out + total, n.flat.data(), n.flat.size() * 4);
      total += static_cast<int64_t>(n.flat.size());
    }
    *n_nets = static_cast<int>(c.nets.size());
    *n_params = total;
    *count = c.count;
    *dim = static_cast<int>(c.mean.size());
    if (mean) std::memcpy(mean, c.mean.data(), c.mean.size() * 8);
    if (m2) std::memcpy(m2, c.m2.data(), c.m2.size() * 8);
  });
}

}  // extern "C"

// ------------------------------------------------ learner / actor checkpoints
// Net names: V-learner "q1", "q2", "q1_target", "q2_target", "policy" (the
// lagged policy); P-learner "policy", "q1", "q2" (the critic replicas);
// actor "policy".  The normalizer block holds the stats the core last
// adopted (the actor: its running normalizer).
#include "../../include/pqlg.h"

struct pqlg_vlearner_s;
struct pqlg_plearner_s;
struct pqlg_actor_s;

namespace pqlg {
VLearner* vlearner_of(pqlg_vlearner h);
PLearner* plearner_of(pqlg_plearner h);
Actor* actor_of(pqlg_actor h);
}  // namespace pqlg

extern "C" {

int pqlg_vlearner_save(pqlg_vlearner h, const char* path) {
  return guarded([&] {
    VLearner& v = *vlearner_of(h);
    File c;
    const char* names[5] = {"q1", "q2", "q1_target", "q2_target", "policy"};
    for (int w = 0; w < 5; ++w) {
      std::vector<float> flat(v.param_count(w));
      v.get_params(w, flat.data());
      c.nets.push_back(make_net(names[w], w == 4 ? v.policy_shape() : v.critic_shape(),
                                std::move(flat)));
    }
    set_norm(c, v.norm_count_, v.norm_mean_, v.norm_m2_, v.obs_dim());
    write(path, c);
  });
}

int pqlg_vlearner_load(pqlg_vlearner h, const char* path) {
  return guarded([&] {
    VLearner& v = *vlearner_of(h);
    const File c = read(path);
    const char* names[5] = {"q1", "q2", "q1_target", "q2_target", "policy"};
    for (int w = 0; w < 5; ++w)
      v.set_params(w, find(c, names[w], w == 4 ? v.policy_shape() : v.critic_shape()).flat.data());
    require(static_cast<int>(c.mean.size()) == v.obs_dim(), "checkpoint: normalizer dim mismatch");
    v.adopt_norm(c.count, c.mean.data(), c.m2.data());
  });
}

int pqlg_plearner_save(pqlg_plearner h, const char* path) {
  return guarded([&] {
    PLearner& p = *plearner_of(h);
    File c;
    const char* names[3] = {"policy", "q1", "q2"};
    for (int w = 0; w < 3; ++w) {
      std::vector<float> flat(p.param_count(w));
      p.get_params(w, flat.data());
      c.nets.push_back(make_net(names[w], w == 0 ? p.policy_shape() : p.critic_shape(),
                                std::move(flat)));
    }
    set_norm(c, p.norm_count_, p.norm_mean_, p.norm_m2_, p.obs_dim());
    write(path, c);
  });
}

int pqlg_plearner_load(pqlg_plearner h, const char* path) {
  return guarded([&] {
    PLearner& p = *plearner_of(h);
    const File c = read(path);
    const char* names[3] = {"policy", "q1", "q2"};
    for (int w = 0; w < 3; ++w)
      p.set_params(w, find(c, names[w], w == 0 ? p.policy_shape() : p.critic_shape()).flat.data());
    require(static_cast<int>(c.mean.size()) == p.obs_dim(), "checkpoint: normalizer dim mismatch");
    p.adopt_norm(c.count, c.mean.data(), c.m2.data());
  });
}

int pqlg_actor_save(pqlg_actor h, const char* path) {
  return guarded([&] {
    Actor& a = *actor_of(h);
    File c;
    std::vector<float> flat(a.param_count());
    a.read_state(5, flat.data());
    c.nets.push_back(make_net("policy", a.policy_shape(), std::move(flat)));
    c.mean.resize(a.obs_dim());
    c.m2.resize(a.obs_dim());
    a.norm(&c.count, c.mean.data(), c.m2.data());
    write(path, c);
  });
}

int pqlg_actor_load(pqlg_actor h, const char* path) {
  return guarded([&] {
    Actor& a = *actor_of(h);
    const File c = read(path);
    const Net& n = find(c, "policy", a.policy_shape());
    a.adopt_policy(n.flat.data(), a.policy_version(), false);
    require(static_cast<int>(c.mean.size()) == a.obs_dim(), "checkpoint: normalizer dim mismatch");
    a.set_norm(c.count, c.mean.data(), c.m2.data());
  });
}

}  // extern "C"
