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

int main(int argc, char **argv) {
  // C4-shaped: Llama-70B, ranks (default 2048) x 8 per host, global batch (default 16384)
  maya_model m{80, 8192, 8192, 128256, 0, 0};
  const int ranks = argc > 1 ? atoi(argv[1]) : 2048;
  const long gbs = argc > 2 ? atol(argv[2]) : 16384;
  maya_cluster cl{ranks / 8, 8, 80ll << 30};
  std::vector<maya_config> cfgs;
  int tps[] = {1, 2, 4, 8}, pps[] = {2, 4, 8, 16}, vss[] = {2, 4, 5, 10};
  const bool big = argc > 3;   // the largest configs only (pp x virtual stages >= 40, micro_mult >= 8)
  for (int tp : tps) for (int pp : pps) for (int mm = big ? 8 : 1; mm <= 16; mm += big ? 4 : 3) for (int vs : vss)
    for (int rc = 1; rc >= 0; rc--) for (int dz = 1; dz >= 0; dz--) {
      if (big && pp * vs < 40) continue;
      maya_config c{tp, pp, mm, vs, rc, 1, dz, 0, gbs};
      GenJob g;
      if (generate_job(m, c, cl, -1, 5000, g, nullptr) == 0) cfgs.push_back(c);
      if (cfgs.size() == 64) goto done;
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
  printf("%zu C4 configs, 1 thread:", cfgs.size()); printf(" generator alone %.1f ms (%zu events, %zu blocks of %zu launches over 3 passes); fused gen+pack %.1f ms\n",
         tgen * 1e3, ns.n / 3, ns.blk / 3, ns.kev / 3, tfull * 1e3);
  const char *nm[] = {"generate_job", "generate_trace", "comm tables", "finish", "pack_tail", "collapse", "slots+wfeats", "rank tables+rcolls", "coll_wf+folded", "renumber_features", "phases packed", "phases replayed", "trace prologue", "trace setup", "pipeline_order", "epilogue+finish"};
  for (int i = 0; i < 16; i++) printf("%-20s %7.3f ms/config\n", nm[i], hp_acc[i] * 1e3 / 9 / cfgs.size());
  return 0;
}
