// Library-level C ABI: error reporting and build information.
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace lk {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static std::atomic<int64_t> g_launches{0};

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LK_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
  return LK_OK;
}

// ------------------------------------------------ test-only path knobs ----
static constexpr int kKnobs = 6;
static std::atomic<int> g_knobs[kKnobs];
static const int kKnobMax[kKnobs] = {1, 1, 1, 1, 3, 1};

int path_knob(int knob) { return (knob >= 0 && knob < kKnobs) ? g_knobs[knob].load(std::memory_order_relaxed) : 0; }

// ---------------------------------------------------------- profiling ----
struct ProfRec {
  int stage;
  cudaEvent_t a, b;
  int64_t launches;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;          // recorded, not yet collected
static std::vector<cudaEvent_t> g_pool;      // free events

static cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

ProfScope::ProfScope(int stage, cudaStream_t st) : stage_(stage), st_(st) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return;
  active_ = true;
  a_ = take_event();
  b_ = take_event();
  mark_ = g_launches.load();
  cudaEventRecord(a_, st_);
}

ProfScope::~ProfScope() {
  if (!active_) return;
  cudaEventRecord(b_, st_);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back({stage_, a_, b_, g_launches.load() - mark_});
}

}  // namespace lk

extern "C" void lk_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(lk::g_prof_mu);
  lk::g_prof_on = on != 0;
}

extern "C" int lk_profile_collect(double* ms4, int64_t* launches4) {
  std::vector<lk::ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(lk::g_prof_mu);
    recs.swap(lk::g_prof);
  }
  for (int i = 0; i < 4; ++i) {
    if (ms4) ms4[i] = 0.0;
    if (launches4) launches4[i] = 0;
  }
  int rc = LK_OK;
  for (auto& r : recs) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess) rc = lk::fail(LK_CUDA_ERROR, cudaGetErrorString(e));
    if (r.stage >= 0 && r.stage < 4) {
      if (ms4) ms4[r.stage] += ms;
      if (launches4) launches4[r.stage] += r.launches;
    }
  }
  std::lock_guard<std::mutex> lk(lk::g_prof_mu);
  for (auto& r : recs) {
    lk::g_pool.push_back(r.a);
    lk::g_pool.push_back(r.b);
  }
  return rc;
}

extern "C" int64_t lk_launch_count(void) { return lk::g_launches.load(); }

extern "C" const char* lk_last_error(void) { return lk::g_last_error.c_str(); }

extern "C" const char* lk_version(void) { return "liger_b200 0.1.0 (sm_100a)"; }

extern "C" int lk_has_tcgen05(void) {
#ifdef LK_HAS_TCGEN05
  return 1;
#else
  return 0;
#endif
}

extern "C" int lk_test_select_path(int knob, int value) {
  if (knob < 0 || knob >= lk::kKnobs || value < 0 || value > lk::kKnobMax[knob]) return -1;
  return lk::g_knobs[knob].exchange(value);
}
