// Multi-threaded host gen+pack timing (mirrors maya_batch_add_generated's worker).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include "../paper_2503_20191_b200/csrc/gen.h"
#include "../paper_2503_20191_b200/csrc/pack.h"
using namespace maya;
int main(int argc, char **argv) {
  int nt = argc > 1 ? atoi(argv[1]) : 8;
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
  for (int it = 0; it < 3; it++) {
    static std::vector<JobPack> packs(512);
    auto t0 = std::chrono::steady_clock::now();
    std::atomic<int> next(0);
    auto work = [&]() {
      GenJob g;
      for (;;) {
        int i = next.fetch_add(1);
        if (i >= (int)cfgs.size()) break;
        generate_job(m, cfgs[i], cl, -1, 5000, g, nullptr);
        maya_raw_job raw = g.raw(0);
        pack_job(raw, i, packs[i], true);
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nt; t++) th.emplace_back(work);
    for (auto &t : th) t.join();
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %d: gen+pack %zu configs %.1f ms\n", nt, cfgs.size(), dt * 1e3);
  }
}
