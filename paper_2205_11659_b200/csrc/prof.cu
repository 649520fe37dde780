// Launch accounting and optional per-kernel CUDA-event timing (used by
// bench.py for the roofline's per-kernel durations; off by default).
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"

namespace tb {
namespace {
std::atomic<long long> g_launches{0};
std::atomic<int> g_prof_on{0};
struct Rec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_mu;
std::vector<Rec> g_pending;
std::vector<cudaEvent_t> g_pool;
std::map<std::string, std::pair<long long, double>> g_acc;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void prof_begin(cudaStream_t s, const char* name, void** token) {
  g_launches.fetch_add(1);
  *token = nullptr;
  if (!g_prof_on.load()) return;
  std::lock_guard<std::mutex> lk(g_mu);
  Rec* r = new Rec{name, get_event(), get_event()};
  cudaEventRecord(r->a, s);
  *token = r;
}

void prof_end(cudaStream_t s, void* token) {
  if (!token) return;
  Rec* r = (Rec*)token;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(r->b, s);
  g_pending.push_back(*r);
  delete r;
}

int sm_count() {  // streaming multiprocessors of the current device (cached per device)
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& c = cache[dev & 63];
  if (c == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    c = v > 0 ? v : 1;
  }
  return c;
}

bool once_per_device(int slot) {
  static std::mutex mu;
  static uint64_t done[16] = {};  // [slot] bit d = done on device d (< 64)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const uint64_t bit = 1ull << (dev & 63);
  if (done[slot & 15] & bit) return false;
  done[slot & 15] |= bit;
  return true;
}

}  // namespace tb

extern "C" {

long long tb_launch_count(void) { return tb::g_launches.load(); }

int tb_profile_enable(int on) {
  tb::g_prof_on.store(on ? 1 : 0);
  return 0;
}

// Fold completed records into per-kernel totals and print them as JSON
// {"kernel": [count, total_ms], ...} into buf; clears the totals.
int tb_profile_read(char* buf, size_t cap) {
  std::lock_guard<std::mutex> lk(tb::g_mu);
  for (auto& r : tb::g_pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& e = tb::g_acc[r.name];
    e.first += 1;
    e.second += ms;
    tb::g_pool.push_back(r.a);
    tb::g_pool.push_back(r.b);
  }
  tb::g_pending.clear();
  std::string s = "{";
  bool first = true;
  for (auto& kv : tb::g_acc) {
    char tmp[256];
    snprintf(tmp, sizeof tmp, "%s\"%s\": [%lld, %.6f]", first ? "" : ", ", kv.first.c_str(), kv.second.first,
             kv.second.second);
    s += tmp;
    first = false;
  }
  s += "}";
  tb::g_acc.clear();
  if (buf && cap) {
    snprintf(buf, cap, "%s", s.c_str());
  }
  return (int)s.size();
}

}  // extern "C"
