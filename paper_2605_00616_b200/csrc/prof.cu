// prof.cu -- launch counter and CUDA-event kernel timing (emu_profile_* ABI).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "emu_internal.cuh"
#include "prof.h"

namespace emu {

static std::atomic<long long> g_launches{0};
static std::atomic<bool> g_prof{false};
static std::mutex g_mu;
struct Acc {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  double ms = 0;
  long long n = 0;
};
static std::map<std::string, Acc>* g_acc = new std::map<std::string, Acc>();
static std::vector<cudaEvent_t>* g_free = new std::vector<cudaEvent_t>();

static cudaEvent_t take_event() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_free->empty()) {
    cudaEvent_t e = g_free->back();
    g_free->pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void prof_count() { g_launches.fetch_add(1, std::memory_order_relaxed); }
bool prof_on() { return g_prof.load(std::memory_order_relaxed); }
void prof_begin(cudaStream_t s, cudaEvent_t* a) {
  *a = take_event();
  cudaEventRecord(*a, s);
}
void prof_end(const char* name, cudaStream_t s, cudaEvent_t a) {
  cudaEvent_t b = take_event();
  cudaEventRecord(b, s);
  std::lock_guard<std::mutex> lk(g_mu);
  (*g_acc)[name].pending.emplace_back(a, b);
}

}  // namespace emu

using namespace emu;

extern "C" {

int64_t emu_launch_count(void) { return g_launches.load(); }

int emu_profile_enable(int on) {
  g_prof.store(on != 0);
  return EMU_OK;
}

int emu_profile_read(const char* kernel, double* total_ms, int64_t* launches) {
  if (!kernel) return fail(EMU_ERR_INVALID, "kernel name is NULL");
  EMU_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_mu);
  Acc& a = (*g_acc)[kernel];
  for (auto& pr : a.pending) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
      a.ms += ms;
      a.n += 1;
    }
    g_free->push_back(pr.first);
    g_free->push_back(pr.second);
  }
  a.pending.clear();
  if (total_ms) *total_ms = a.ms;
  if (launches) *launches = a.n;
  a.ms = 0;
  a.n = 0;
  return EMU_OK;
}

// Newline-separated names of every kernel with launches recorded since they
// were last read (emu_profile_read), truncated to cap - 1 bytes.
int emu_profile_names(char* buf, int64_t cap) {
  if (!buf || cap < 1) return fail(EMU_ERR_INVALID, "buffer is NULL or empty");
  std::string out;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : *g_acc)
      if (!kv.second.pending.empty() || kv.second.n) out += kv.first + "\n";
  }
  const size_t n = std::min<size_t>(out.size(), (size_t)cap - 1);
  memcpy(buf, out.data(), n);
  buf[n] = 0;
  return EMU_OK;
}

}  // extern "C"
