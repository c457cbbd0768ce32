// Launch tracing: per-launch device durations from CUDA events recorded on the launching stream
// (regen_trace_enable / regen_trace_read in include/regen.h). Used by bench.py to time the dominant
// kernel live inside the timed region; off by default.
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace regen {

namespace {
struct Rec {
  const char* name;
  cudaEvent_t e0, e1;
};
std::atomic<bool> g_on{false};
char g_filter[REGEN_TRACE_NAME_LEN] = "";   // only names starting with it ("" = all)
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// Inside a stream capture a plain event record only orders work within the graph; the external
// flag makes the graph record the event for real on every launch, so it can be timed.
void record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else cudaEventRecord(e, s);
}
}  // namespace

bool trace_on() { return g_on.load(std::memory_order_relaxed); }

void trace_begin(const char* name, cudaStream_t s, int* slot) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_filter[0] && strncmp(name, g_filter, strlen(g_filter)) != 0) return;
  Rec r;
  r.name = name;
  r.e0 = take_event();
  r.e1 = take_event();
  record(r.e0, s);
  g_recs.push_back(r);
  *slot = (int)g_recs.size() - 1;
}

void trace_end(int slot, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (slot < (int)g_recs.size()) record(g_recs[slot].e1, s);
}

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_trace_enable(int32_t on) {
  g_on.store(on != 0);
  return REGEN_OK;
}

extern "C" regen_status regen_trace_filter(const char* prefix) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (prefix) {
    strncpy(g_filter, prefix, REGEN_TRACE_NAME_LEN - 1);
    g_filter[REGEN_TRACE_NAME_LEN - 1] = 0;
  } else {
    g_filter[0] = 0;
  }
  return REGEN_OK;
}

extern "C" regen_status regen_trace_read(char* names, float* ms, int32_t cap, int32_t* n) {
  REGEN_REQUIRE(n != nullptr, "n is null");
  std::lock_guard<std::mutex> lk(g_mu);
  int32_t k = 0;
  for (auto& r : g_recs) {
    cudaError_t e = cudaEventSynchronize(r.e1);
    if (k < cap) {
      float t = 0.f;
      if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.e0, r.e1);
      if (e != cudaSuccess) {
        t = -(float)e;           // not timed (reported as -cudaError)
        cudaGetLastError();      // do not leave it as the thread's last error
      }
      if (ms) ms[k] = t;
      if (names) {
        strncpy(names + (size_t)k * REGEN_TRACE_NAME_LEN, r.name, REGEN_TRACE_NAME_LEN - 1);
        names[(size_t)k * REGEN_TRACE_NAME_LEN + REGEN_TRACE_NAME_LEN - 1] = 0;
      }
    }
    ++k;
    g_pool.push_back(r.e0);
    g_pool.push_back(r.e1);
  }
  g_recs.clear();
  *n = k;
  return REGEN_OK;
}
