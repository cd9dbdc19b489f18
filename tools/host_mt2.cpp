// Multi-threaded fused gen+pack timing, as maya_batch_add_generated runs it
// (pack_generated with kernel blocks and a shared GenCache, longest first,
// the engine's WorkerPool): wall time and per-thread busy time.
//   g++ -O2 -std=c++17 -Iinclude tools/host_mt2.cpp paper_2503_20191_b200/csrc/{gen,pack}.cpp -lpthread
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include "../paper_2503_20191_b200/csrc/gen.h"
#include "../paper_2503_20191_b200/csrc/pack.h"
#include "../paper_2503_20191_b200/csrc/pool.h"
using namespace maya;
using clk = std::chrono::steady_clock;
int main(int argc, char **argv) {
  maya_model m{24, 2048, 2048, 51200, 0, 0};
  maya_cluster cl{1, 8, 80ll << 30};
  std::vector<maya_config> cfgs;
  int tps[] = {1, 2, 4, 8}, pps[] = {1, 2, 4, 8}, mms[] = {1, 2, 4, 6, 8}, vss[] = {1, 2, 4};
  for (int tp : tps) for (int pp : pps) for (int mm : mms) for (int vs : vss)
    for (int rc = 1; rc >= 0; rc--) for (int sp = 1; sp >= 0; sp--) for (int dz = 1; dz >= 0; dz--) {
      maya_config c{tp, pp, mm, vs, rc, sp, dz, 0, 512};
      GenJob g;
      if (generate_job(m, c, cl, -1, 5000, g, nullptr) == 0) cfgs.push_back(c);
      if (cfgs.size() == 512) goto done;
    }
done:
  const int n = (int)cfgs.size();
  std::vector<int> lpt(n);
  for (int i = 0; i < n; i++) lpt[i] = i;
  auto cost = [&](int i) { return (long)cfgs[i].pp * cfgs[i].micro_mult * std::max(1, cfgs[i].virtual_stages); };
  std::stable_sort(lpt.begin(), lpt.end(), [&](int a, int b) { return cost(a) > cost(b); });
  static std::vector<JobPack> packs(512);
  for (int a = 1; a < argc; a++) {
    const int nt = atoi(argv[a]);
    for (int it = 0; it < 4; it++) {
      std::atomic<int> next(0);
      std::vector<double> busy(64, 0.0);
      std::atomic<int> tid(0);
      GenCache cache;
      auto t0 = clk::now();
      auto work = [&]() {
        thread_local GenJob g;
        const int me = tid.fetch_add(1);
        auto b0 = clk::now();
        for (;;) {
          int q = next.fetch_add(1);
          if (q >= n) break;
          const int i = lpt[q];
          std::string err;
          packs[i].clear();
          pack_generated(m, cfgs[i], cl, -1, 5000, 0, i, true, g, packs[i], &err, true, &cache);
        }
        busy[me] = std::chrono::duration<double>(clk::now() - b0).count();
      };
      WorkerPool::get().run(nt, work);
      double dt = std::chrono::duration<double>(clk::now() - t0).count();
      double mx = 0, sum = 0;
      for (int t = 0; t < nt; t++) { mx = std::max(mx, busy[t]); sum += busy[t]; }
      if (it == 3)
        printf("threads %2d: wall %.2f ms, busy max %.2f mean %.2f ms, thread-sum %.1f ms\n", nt,
               dt * 1e3, mx * 1e3, sum / nt * 1e3, sum * 1e3);
    }
  }
}
