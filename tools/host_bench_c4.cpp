// Host-only timing of fused generate + pack for C4-shaped configs (one core):
//   g++ -O2 -std=c++17 -Iinclude tools/host_bench_c4.cpp paper_2503_20191_b200/csrc/{gen,pack}.cpp -lpthread
//   ./a.out [ranks] [global_batch]
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../paper_2503_20191_b200/csrc/gen.h"
#include "../paper_2503_20191_b200/csrc/pack.h"
using namespace maya;
using clk = std::chrono::steady_clock;
int main(int argc, char **argv) {
  maya_model m{80, 8192, 8192, 128256, 0, 0};
  int ranks = argc > 1 ? atoi(argv[1]) : 2048;
  long gb = argc > 2 ? atol(argv[2]) : 4096;
  maya_cluster cl{ranks / 8, 8, 80ll << 30};
  std::vector<maya_config> cfgs;
  int tps[] = {1, 2, 4, 8}, pps[] = {2, 4, 8, 16}, vss[] = {2, 4, 5, 10};
  for (int tp : tps) for (int pp : pps) for (int mm = 1; mm <= 16; mm++) for (int vs : vss)
    for (int rc = 1; rc >= 0; rc--) for (int dz = 1; dz >= 0; dz--) {
      maya_config c{tp, pp, mm, vs, rc, 1, dz, 0, gb};
      GenJob g;
      if (generate_job(m, c, cl, -1, 5000, g, nullptr) == 0) cfgs.push_back(c);
      if (cfgs.size() == 64) goto done;
    }
done:
  double best = 1e9; size_t recs = 0, ev = 0;
  for (int it = 0; it < 3; it++) {
    double t = 0; recs = 0; ev = 0;
    GenJob g;
    for (auto &c : cfgs) {
      JobPack P; std::string err;
      auto a = clk::now();
      pack_generated(m, c, cl, -1, 5000, 0, 0, true, g, P, &err, true);
      t += std::chrono::duration<double>(clk::now() - a).count();
      recs += P.ops.size();
      for (auto &h : P.reps) ev += h.n_events;
    }
    best = std::min(best, t);
  }
  printf("%zu configs at %d ranks gb %ld: fused gen+pack %.1f ms (%.2f ms/config), %zu rep events, %zu op records\n",
         cfgs.size(), ranks, gb, best * 1e3, best * 1e3 / cfgs.size(), ev, recs);
}
