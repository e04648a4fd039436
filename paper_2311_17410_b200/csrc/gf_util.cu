// gf_util.cu -- error state, version, launch counter, seed helpers.
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <vector>

#include "gf_common.cuh"

namespace gf {
static thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_profile{0};

thread_local std::string g_prof_tag;

struct ProfRec {
  std::string name;
  cudaEvent_t e0, e1;
};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;

cudaEvent_t prof_start(cudaStream_t s) {
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  cudaEventRecord(e, s);
  return e;
}
void prof_stop(const char* name, cudaStream_t s, cudaEvent_t e0) {
  cudaEvent_t e1 = nullptr;
  if (cudaEventCreate(&e1) != cudaSuccess) return;
  cudaEventRecord(e1, s);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back({g_prof_tag.empty() ? std::string(name) : std::string(name) + "[" + g_prof_tag + "]", e0, e1});
}
static void prof_clear() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  g_prof.clear();
}

void set_error(const std::string& msg) { t_err = msg; }
gf_status fail(gf_status st, const std::string& msg) {
  t_err = msg;
  return st;
}

// numpy.random.SeedSequence (pool size 4, 32-bit words), the algorithm behind
// reference hop_seed (sampling.py:135-137).
static uint32_t ss_hashmix(uint32_t value, uint32_t* hc) {
  value ^= *hc;
  *hc *= 0x931e8875u;
  value *= *hc;
  value ^= value >> 16;
  return value;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}
static int ss_words(uint64_t v, uint32_t* out) {
  int n = 0;
  if (v == 0) {
    out[n++] = 0;
    return n;
  }
  while (v) {
    out[n++] = (uint32_t)v;
    v >>= 32;
  }
  return n;
}
uint64_t seed_sequence_2(uint64_t a, uint64_t b) {
  uint32_t ent[8];
  int ne = ss_words(a, ent);
  ne += ss_words(b, ent + ne);
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < ne ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < ne; s++)
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
  uint32_t st[2];
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < 2; i++) {
    uint32_t x = pool[i];
    x ^= hb;
    hb *= 0x58f38dedu;
    x *= hb;
    x ^= x >> 16;
    st[i] = x;
  }
  return (uint64_t)st[0] | ((uint64_t)st[1] << 32);
}
}  // namespace gf

extern "C" {
const char* gf_last_error(void) { return gf::t_err.c_str(); }
const char* gf_version(void) { return "gfb200 0.1.0 (sm_100a)"; }
uint64_t gf_launch_count(void) { return gf::g_launches.load(); }
void gf_profile_enable(int on) {
  gf::prof_clear();
  gf::g_profile.store(on ? 1 : 0);
}
gf_status gf_profile_summary(char* buf, int64_t len) {
  if (!buf || len <= 0) return gf::fail(GF_EINVAL, "NULL buffer");
  cudaDeviceSynchronize();
  std::map<std::string, std::pair<int64_t, double>> agg;
  {
    std::lock_guard<std::mutex> lk(gf::g_prof_mu);
    for (auto& r : gf::g_prof) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.e0, r.e1);
      auto& a = agg[r.name];
      a.first += 1;
      a.second += ms;
    }
  }
  std::string out;
  char line[512];
  for (auto& kv : agg) {
    snprintf(line, sizeof(line), "%s\t%lld\t%.6f\n", kv.first.c_str(), (long long)kv.second.first, kv.second.second);
    out += line;
  }
  if ((int64_t)out.size() + 1 > len) return gf::fail(GF_ERANGE, "profile buffer too small");
  memcpy(buf, out.c_str(), out.size() + 1);
  return GF_OK;
}
uint64_t gf_hop_seed(uint64_t seed, uint64_t hop) { return gf::seed_sequence_2(seed, hop); }
uint64_t gf_child_key(uint64_t parent, uint64_t j) { return gf::child_key(parent, j); }
}
