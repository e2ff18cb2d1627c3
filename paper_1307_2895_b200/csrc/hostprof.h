// Sampling profiler of the host thread running hifde_factor (diagnostics
// only, HIFDE_SAMPLE=<file>): a timer thread signals the factor thread every
// 50 us; the handler records its call stack; the raw return addresses (as
// offsets into this library) are written at the end of the factorization and
// symbolized offline (tools/hostprof_report.py, addr2line).
#pragma once
namespace hifde {
void host_sampler_start();
void host_sampler_stop(const char* path);
}  // namespace hifde
