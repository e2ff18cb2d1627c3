#include "hostprof.h"

#include <dlfcn.h>
#include <execinfo.h>
#include <pthread.h>
#include <signal.h>
#include <time.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <thread>

namespace hifde {
namespace {
constexpr int kDepth = 24;
constexpr int kMax = 1 << 16;
void* g_frames[kMax][kDepth];
int g_depth[kMax];
std::atomic<int> g_n{0};
std::atomic<bool> g_run{false};
pthread_t g_target;
std::thread g_timer;

void on_prof(int) {
  const int i = g_n.fetch_add(1);
  if (i >= kMax) return;
  g_depth[i] = backtrace(g_frames[i], kDepth);
}
}  // namespace

void host_sampler_start() {
  void* warm[4];
  backtrace(warm, 4);  // load the unwinder outside the handler
  struct sigaction sa {};
  sa.sa_handler = on_prof;
  sa.sa_flags = SA_RESTART;
  sigaction(SIGPROF, &sa, nullptr);
  g_n = 0;
  g_target = pthread_self();
  g_run = true;
  g_timer = std::thread([]() {
    timespec ts{0, 700000};  // ~1 kHz: low enough not to perturb the threads
    while (g_run.load()) {
      pthread_kill(g_target, SIGPROF);
      nanosleep(&ts, nullptr);
    }
  });
}

void host_sampler_stop(const char* path) {
  g_run = false;
  if (g_timer.joinable()) g_timer.join();
  Dl_info info{};
  dladdr((void*)&host_sampler_start, &info);
  const uintptr_t base = (uintptr_t)info.dli_fbase;
  FILE* fp = fopen(path, "a");  // accumulate over factorizations
  if (!fp) return;
  const int n = g_n.load() < kMax ? g_n.load() : kMax;
  fprintf(fp, "# base %p lib %s samples %d\n", (void*)base, info.dli_fname ? info.dli_fname : "?", n);
  for (int i = 0; i < n; ++i) {
    for (int d = 0; d < g_depth[i]; ++d) {
      const uintptr_t a = (uintptr_t)g_frames[i][d];
      Dl_info fi{};
      const bool ours = dladdr(g_frames[i][d], &fi) && fi.dli_fbase == info.dli_fbase;
      if (ours) fprintf(fp, " %lx", (unsigned long)(a - base));
      else fprintf(fp, " x");
    }
    fprintf(fp, "\n");
  }
  fclose(fp);
}

}  // namespace hifde
