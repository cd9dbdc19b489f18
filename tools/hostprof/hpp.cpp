// Host-only breakdown of the fused generate+pack path (no GPU needed):
// generator alone (a sink that takes blocks and does nothing), full fused
// pack_generated, and the share of pack_tail (collapse + tables).
//   g++ -O2 -std=c++17 tools/host_prof.cpp paper_2503_20191_b200/csrc/{gen,pack}.cpp -lpthread
#include <chrono>
#include <cstdio>
#include <vector>

#include "/tmp/hprof/gen.h"
#include "/tmp/hprof/pack.h"

using namespace maya;
namespace maya { extern double hp_acc[16]; }
using clk = std::chrono::steady_clock;

struct NullSink final : EventSink {
  size_t n = 0, blk = 0, kev = 0;
  void rep_begin(size_t) override {}
  void ev(uint8_t, int32_t, int64_t, int64_t, int64_t, int64_t) override { n++; }
  void rep_end() override {}
  bool takes_blocks() const override { return true; }
  uint32_t kernel_block(int32_t, const KSpec *, size_t k, int64_t, int32_t) override { blk++; kev += k; return ~0u; }
};

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
  for (int q = 0; q < 16; q++) hp_acc[q] = 0;   // only the timed passes
  GenJob g;
  NullSink ns;
  double tgen = 0, tfull = 0;
  for (int it = 0; it < 9; it++) {
    auto t0 = clk::now();
    
    auto t1 = clk::now();
    GenCache cache;   // one per batch, as maya_batch_add_generated
    for (auto &c : cfgs) {
      JobPack P;
      std::string err;
      pack_generated(m, c, cl, -1, 5000, 0, 0, true, g, P, &err, true, &cache);
    }
    auto t2 = clk::now();
    tgen = it ? std::min(tgen, std::chrono::duration<double>(t1 - t0).count()) : std::chrono::duration<double>(t1 - t0).count();
    tfull = it ? std::min(tfull, std::chrono::duration<double>(t2 - t1).count()) : std::chrono::duration<double>(t2 - t1).count();
  }
  printf("512 configs, 1 thread: generator alone %.1f ms (%zu events, %zu blocks of %zu launches over 3 passes); fused gen+pack %.1f ms\n",
         tgen * 1e3, ns.n / 3, ns.blk / 3, ns.kev / 3, tfull * 1e3);
  const char *nm[] = {"generate_job", "generate_trace", "comm tables", "finish", "pack_tail", "collapse", "slots+wfeats", "rank tables+rcolls", "coll_wf+folded", "renumber_features", "phases packed", "phases replayed", "trace prologue", "trace setup", "pipeline_order", "epilogue+finish"};
  for (int i = 0; i < 16; i++) printf("%-20s %7.1f ms/pass\n", nm[i], hp_acc[i] * 1e3 / 9);
  return 0;
}
