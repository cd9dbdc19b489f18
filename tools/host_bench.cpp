// Host-only timing of trace generation and SoA packing (no GPU needed).
//   g++ -O2 -std=c++17 tools/host_bench.cpp paper_2503_20191_b200/csrc/{gen,pack}.cpp -lpthread
#include <chrono>
#include <cstdio>
#include <vector>

#include "../paper_2503_20191_b200/csrc/gen.h"
#include "../paper_2503_20191_b200/csrc/pack.h"

using namespace maya;
using clk = std::chrono::steady_clock;

int main() {
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
  double tg = 0, tp = 0;
  size_t ev = 0;
  for (int it = 0; it < 2; it++) {
    tg = tp = 0;
    ev = 0;
    for (auto &c : cfgs) {
      GenJob g;
      auto t0 = clk::now();
      generate_job(m, c, cl, -1, 5000, g, nullptr);
      auto t1 = clk::now();
      maya_raw_job raw = g.raw(0);
      JobPack P;
      pack_job(raw, 0, P, true);
      auto t2 = clk::now();
      tg += std::chrono::duration<double>(t1 - t0).count();
      tp += std::chrono::duration<double>(t2 - t1).count();
      ev += g.ev_kind.size();
    }
  }
  printf("%zu configs, %zu events: gen %.1f ms (%.1f ns/ev), pack %.1f ms (%.1f ns/ev)\n",
         cfgs.size(), ev, tg * 1e3, tg * 1e9 / ev, tp * 1e3, tp * 1e9 / ev);
  double tf = 0;
  for (int it = 0; it < 2; it++) {
    tf = 0;
    GenJob g;
    for (auto &c : cfgs) {
      JobPack P;
      std::string err;
      auto t0 = clk::now();
      pack_generated(m, c, cl, -1, 5000, 0, 0, true, g, P, &err);
      tf += std::chrono::duration<double>(clk::now() - t0).count();
    }
  }
  printf("fused generate+pack %.1f ms (%.1f ns/ev)\n", tf * 1e3, tf * 1e9 / ev);
  size_t recs = 0, blks = 0, bf = 0, ops0 = 0;
  for (int it = 0; it < 2; it++) {
    tf = 0;
    recs = blks = bf = ops0 = 0;
    GenJob g;
    for (auto &c : cfgs) {
      JobPack P;
      std::string err;
      auto t0 = clk::now();
      pack_generated(m, c, cl, -1, 5000, 0, 0, true, g, P, &err, true);
      tf += std::chrono::duration<double>(clk::now() - t0).count();
      recs += P.ops.size();
      blks += P.blocks.size();
      bf += P.blk_fids.size();
    }
  }
  printf("fused generate+pack, kernel blocks %.1f ms (%.1f ns/ev): %zu op records, %zu blocks, "
         "%zu block fids\n", tf * 1e3, tf * 1e9 / ev, recs, blks, bf);
  return 0;
}
