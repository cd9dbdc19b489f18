// Phase-template replay and the per-batch layout cache (GenCache) must not
// change a packed job: pack_generated in kernel-block mode with templates and
// cache on, and with both off, byte-compared, over the C2 lattice, small
// lattices on every schedule and odd overheads.
//   g++ -O2 -std=c++17 tools/replay_check.cpp paper_2503_20191_b200/csrc/{gen,pack}.cpp -lpthread
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_2503_20191_b200/csrc/gen.h"
#include "../paper_2503_20191_b200/csrc/pack.h"

using namespace maya;
template <typename T>
static bool veq(const std::vector<T> &a, const std::vector<T> &b) {
  return a.size() == b.size() && (a.empty() || !memcmp(a.data(), b.data(), a.size() * sizeof(T)));
}
static bool same(const JobPack &a, const JobPack &b) {
  return !memcmp(&a.hdr, &b.hdr, sizeof a.hdr) && veq(a.reps, b.reps) && veq(a.ops, b.ops) &&
         veq(a.streams, b.streams) && veq(a.stream_events, b.stream_events) &&
         veq(a.coll_lc, b.coll_lc) && veq(a.coll_idx, b.coll_idx) && veq(a.coll_wf, b.coll_wf) &&
         veq(a.syncs, b.syncs) && veq(a.counts, b.counts) && veq(a.mems, b.mems) &&
         veq(a.feats, b.feats) && veq(a.feat_meta, b.feat_meta) && veq(a.blocks, b.blocks) &&
         veq(a.blk_fids, b.blk_fids) && veq(a.comms, b.comms) && veq(a.wfeats, b.wfeats) &&
         veq(a.ranks, b.ranks) && veq(a.rank_comm, b.rank_comm) && veq(a.rcolls, b.rcolls) &&
         veq(a.comm_rdv, b.comm_rdv) && veq(a.rank_orig, b.rank_orig);
}

static int check(const maya_model &m, const maya_cluster &cl, const std::vector<maya_config> &cfgs,
                 int sched, int64_t ovh, double *t_on, double *t_off) {
  int bad = 0;
  GenJob g;
  GenCache cache;
  for (const maya_config &c : cfgs) {
    JobPack a, b;
    std::string e1, e2;
    g_phase_replay = true;
    auto t0 = std::chrono::steady_clock::now();
    int r1 = pack_generated(m, c, cl, sched, ovh, 0, 0, true, g, a, &e1, true, &cache);
    auto t1 = std::chrono::steady_clock::now();
    g_phase_replay = false;
    int r2 = pack_generated(m, c, cl, sched, ovh, 0, 0, true, g, b, &e2, true);
    auto t2 = std::chrono::steady_clock::now();
    *t_on += std::chrono::duration<double>(t1 - t0).count();
    *t_off += std::chrono::duration<double>(t2 - t1).count();
    if (r1 != r2 || (r1 == 0 && !same(a, b))) {
      bad++;
      if (bad < 5) printf("mismatch tp%d pp%d mm%d vs%d rc%d sp%d dz%d gb%lld sched %d\n", c.tp, c.pp,
                          c.micro_mult, c.virtual_stages, c.act_recompute, c.seq_parallel,
                          c.dist_optimizer, (long long)c.global_batch, sched);
    }
  }
  return bad;
}

int main() {
  double on = 0, off = 0;
  int bad = 0, n = 0;
  {
    maya_model m{24, 2048, 2048, 51200, 0, 0};
    maya_cluster cl{1, 8, 80ll << 30};
    std::vector<maya_config> cfgs;
    int tps[] = {1, 2, 4, 8}, pps[] = {1, 2, 4, 8}, mms[] = {1, 2, 4, 6, 8}, vss[] = {1, 2, 4};
    for (int tp : tps) for (int pp : pps) for (int mm : mms) for (int vs : vss)
      for (int rc = 1; rc >= 0; rc--) for (int sp = 1; sp >= 0; sp--) for (int dz = 1; dz >= 0; dz--)
        cfgs.push_back(maya_config{tp, pp, mm, vs, rc, sp, dz, 0, 512});
    bad += check(m, cl, cfgs, -1, 5000, &on, &off);
    n += (int)cfgs.size();
  }
  {  // small model, two hosts, every schedule, odd overheads
    maya_model m{8, 128, 64, 512, 0, 0};
    maya_cluster cl{2, 8, 1ll << 34};
    std::vector<maya_config> cfgs;
    for (int tp : {1, 2, 4}) for (int pp : {1, 2, 4, 8}) for (int mm : {1, 2, 3}) for (int vs : {1, 2})
      for (int rc : {0, 1}) for (int sp : {0, 1}) for (int dz : {0, 1})
        cfgs.push_back(maya_config{tp, pp, mm, vs, rc, sp, dz, 0, 64});
    for (int sched : {-1, 0, 1, 2})
      for (int64_t ovh : {0ll, 777ll}) {
        bad += check(m, cl, cfgs, sched, ovh, &on, &off);
        n += (int)cfgs.size();
      }
  }
  {  // C3 / C4 shapes at 64-2,048 ranks (a sample of each lattice)
    maya_model c3{40, 6144, 2048, 51200, 0, 0}, c4{80, 8192, 8192, 128256, 0, 0};
    for (int ranks : {64, 256, 1024, 2048}) {
      maya_cluster cl{ranks / 8, 8, 80ll << 30};
      for (int which = 0; which < 2; which++) {
        const maya_model &m = which ? c4 : c3;
        std::vector<maya_config> cfgs;
        int k = 0;
        for (int tp : {1, 2, 4, 8}) for (int pp : {1, 2, 4, 8, 16}) for (int mm : {1, 3, 8})
          for (int vs : {1, 2, 4, 5, 10}) for (int rc : {0, 1}) for (int dz : {0, 1}) {
            if ((k++ % 7) != 0) continue;
            maya_config c{tp, pp, mm, vs, rc, which ? 1 : rc, dz, 0, which ? 4096 : 2048};
            GenJob g;
            if (generate_job(m, c, cl, -1, 5000, g, nullptr) == 0) cfgs.push_back(c);
          }
        bad += check(m, cl, cfgs, -1, 5000, &on, &off);
        n += (int)cfgs.size();
      }
    }
  }
  printf("%d packs compared, %d mismatches; replay %.1f ms, event-by-event %.1f ms\n", n, bad,
         on * 1e3, off * 1e3);
  return bad != 0;
}
