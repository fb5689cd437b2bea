// Per-stage device-time accounting for bench.py (vc_profile_* in the C ABI).
// Only active when enabled; it synchronises the stream at the end of every
// block forward, so it is never on the timed path.
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "vc_kernels.h"

namespace vc {

namespace {
struct Stage {
  std::string name;
  double ms = 0;
  int calls = 0;
};
struct Prof {
  bool on = false;
  std::vector<Stage> stages;
  std::vector<cudaEvent_t> events;  // pool
  std::vector<std::string> marks;   // names of the marks of the current call
  cudaStream_t stream = nullptr;
  std::mutex mu;
};
Prof& prof() {
  static Prof p;
  return p;
}
cudaEvent_t pool_event(Prof& p, size_t i) {
  while (p.events.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    p.events.push_back(e);
  }
  return p.events[i];
}
}  // namespace

bool profile_on() { return prof().on; }

void profile_begin(cudaStream_t st) {
  Prof& p = prof();
  if (!p.on) return;
  p.marks.clear();
  p.stream = st;
  cudaEventRecord(pool_event(p, 0), st);
}

void profile_mark(cudaStream_t st, const char* name) {
  Prof& p = prof();
  if (!p.on) return;
  p.marks.push_back(name);
  cudaEventRecord(pool_event(p, p.marks.size()), st);
}

void profile_end() {
  Prof& p = prof();
  if (!p.on || p.marks.empty()) return;
  cudaEventSynchronize(p.events[p.marks.size()]);
  std::lock_guard<std::mutex> g(p.mu);
  for (size_t i = 0; i < p.marks.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.events[i], p.events[i + 1]);
    Stage* s = nullptr;
    for (auto& x : p.stages)
      if (x.name == p.marks[i]) s = &x;
    if (!s) {
      p.stages.push_back(Stage{p.marks[i]});
      s = &p.stages.back();
    }
    s->ms += ms;
    s->calls += 1;
  }
  p.marks.clear();
}

}  // namespace vc

extern "C" {

int vc_profile_enable(int on) {
  vc::prof().on = on != 0;
  return VC_OK;
}

void vc_profile_reset(void) {
  std::lock_guard<std::mutex> g(vc::prof().mu);
  vc::prof().stages.clear();
}

int vc_profile_read(double* ms_total, int32_t* calls, int32_t max_stages, char* names_buf,
                    size_t names_len) {
  auto& p = vc::prof();
  std::lock_guard<std::mutex> g(p.mu);
  std::string names;
  int n = 0;
  for (auto& s : p.stages) {
    if (n >= max_stages) break;
    if (ms_total) ms_total[n] = s.ms;
    if (calls) calls[n] = s.calls;
    if (n) names += "\n";
    names += s.name;
    ++n;
  }
  if (names_buf && names_len) {
    strncpy(names_buf, names.c_str(), names_len - 1);
    names_buf[names_len - 1] = 0;
  }
  return n;
}

}  // extern "C"
