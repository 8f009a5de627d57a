// prof.cuh — optional per-phase device timing (CUTBDDC_PROFILE=1).
//
// Scopes record CUDA events on the handle stream around a launch group; the
// totals per name are printed to stderr when the handle is destroyed. Used to
// find where setup and the solve sweeps spend their time without a profiler
// (nsys is not in the image; ncu serialises launches). Never active inside a
// stream capture.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

namespace cutbddc_b200 {

struct Prof {
  bool on = false;
  struct Rec {
    std::string name;
    cudaEvent_t a, b;
    double host_ms;     // host wall time spent inside the scope (enqueue + host work)
    double host_start;  // host ms since the first scope (timeline mode)
  };
  bool timeline = false;  // CUTBDDC_PROFILE=2: also print every scope in order
  cudaEvent_t base = nullptr;
  std::chrono::steady_clock::time_point hbase;
  std::vector<Rec> pending;
  std::map<std::string, std::pair<long long, double>> tot;  // name -> (count, ms)
  std::map<std::string, double> mx;                         // name -> max ms of one scope
  std::map<std::string, double> host;                       // name -> host ms

  Prof() {
    const char* e = std::getenv("CUTBDDC_PROFILE");
    on = e && (e[0] == '1' || e[0] == '2');
    timeline = e && e[0] == '2';
  }
  void flush() {
    for (auto& r : pending) {
      cudaEventSynchronize(r.b);
      float ms = 0;
      cudaEventElapsedTime(&ms, r.a, r.b);
      if (timeline && base) {  // device start / duration and host start, ms from the first scope
        float st = 0;
        cudaEventElapsedTime(&st, base, r.a);
        std::fprintf(stderr, "[cutbddc timeline] %-40s dev %9.3f +%8.3f  host %9.3f +%8.3f\n", r.name.c_str(), st, ms,
                     r.host_start, r.host_ms);
      }
      auto& t = tot[r.name];
      t.first += 1;
      t.second += ms;
      mx[r.name] = std::max(mx[r.name], (double)ms);
      host[r.name] += r.host_ms;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    pending.clear();
  }
  void dump() {
    if (!on) return;
    flush();
    double all = 0;
    for (auto& kv : tot) all += kv.second.second;
    std::fprintf(stderr, "[cutbddc profile] %-40s %8s %10s %10s %10s %12s\n", "scope", "count", "total ms", "mean us",
                 "max us", "host mean us");
    for (auto& kv : tot)
      std::fprintf(stderr, "[cutbddc profile] %-40s %8lld %10.3f %10.2f %10.2f %12.2f\n", kv.first.c_str(),
                   kv.second.first, kv.second.second, 1e3 * kv.second.second / (double)kv.second.first,
                   1e3 * mx[kv.first], 1e3 * host[kv.first] / (double)kv.second.first);
    std::fprintf(stderr, "[cutbddc profile] (scopes may nest; sum of all = %.3f ms)\n", all);
  }
  ~Prof() {
    for (auto& r : pending) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  }
};

// RAII scope: no-op unless profiling is on and the stream is not capturing.
struct ProfScope {
  Prof* p = nullptr;
  cudaStream_t s = nullptr;
  std::string name;
  cudaEvent_t a = nullptr;
  std::chrono::steady_clock::time_point t0;
  ProfScope(Prof& prof, cudaStream_t st, std::string nm) {
    if (!prof.on) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone) return;
    p = &prof;
    s = st;
    name = std::move(nm);
    cudaEventCreate(&a);
    cudaEventRecord(a, s);
    t0 = std::chrono::steady_clock::now();
    if (prof.timeline && !prof.base) {
      cudaEventCreate(&prof.base);
      cudaEventRecord(prof.base, s);
      prof.hbase = t0;
    }
  }
  void close() {
    if (!p || !a) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, s);
    const double hm = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    p->pending.push_back({name, a, b, hm, std::chrono::duration<double, std::milli>(t0 - p->hbase).count()});
    if (p->pending.size() > 4096) p->flush();
    a = nullptr;
  }
  // close this scope and open the next phase under a new name
  void next(std::string nm) {
    if (!p) return;
    close();
    name = std::move(nm);
    cudaEventCreate(&a);
    cudaEventRecord(a, s);
    t0 = std::chrono::steady_clock::now();
  }
  ~ProfScope() {
    if (p && a) close();
  }
};

}  // namespace cutbddc_b200
