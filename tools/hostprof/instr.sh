set -e
mkdir -p /tmp/hprof && cp /root/repo/paper_2503_20191_b200/csrc/{gen.cpp,pack.cpp,gen.h,pack.h,soa.h,pool.h} /tmp/hprof/ && sed -i 's@#include "../../include/maya_b200.h"@#include "/root/repo/include/maya_b200.h"@' /tmp/hprof/*.h /tmp/hprof/*.cpp
python3 - <<'EOF'
hdr='''#include <chrono>
namespace maya { extern double hp_acc[16]; }
struct HPScope { int i; std::chrono::steady_clock::time_point t0; HPScope(int i_):i(i_),t0(std::chrono::steady_clock::now()){} ~HPScope(){ maya::hp_acc[i]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-t0).count(); } };
#define HPC(a,b) a##b
#define HPX(a,b) HPC(a,b)
#define HP(i) HPScope HPX(hps_, __LINE__)(i)
'''
def rep(s,a,b):
    if a not in s: print("MISSING", a[:60]); return s
    return s.replace(a,b,1)
g=open('/tmp/hprof/gen.cpp').read()
g=rep(g,'#include "gen.h"','#include "gen.h"\n'+hdr)
g=rep(g,"""  G.clear();   // keep capacity: a worker thread reuses one GenJob across configs
  try {""","""  HP(0);
  G.clear();   // keep capacity: a worker thread reuses one GenJob across configs
  try {""")
g=rep(g,"""    G.rank_rep.resize(n);""","""    HP(2);
    G.rank_rep.resize(n);""")
g=rep(g,"""                    int64_t rank, int64_t overhead, int32_t dtype, GenJob &G, RepCalls &rc,
                    EventSink *sink, JobTpls *jtpl) {""","""                    int64_t rank, int64_t overhead, int32_t dtype, GenJob &G, RepCalls &rc,
                    EventSink *sink, JobTpls *jtpl) {
  HP(1);""")
g=rep(g,"""    if (replay && bt.id >= 0 && sink->phase_replay(bt.id, B.next_alloc)) {""","""    auto tph = std::chrono::steady_clock::now();
    if (replay && bt.id >= 0 && sink->phase_replay(bt.id, B.next_alloc)) {""")
g=rep(g,"""        B.last_version[e.first] = B.next_version[e.first] - 1;
      }
      continue;
    }""","""        B.last_version[e.first] = B.next_version[e.first] - 1;
      }
      maya::hp_acc[11]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-tph).count();
      continue;
    }""")
g=rep(g,"""        if (B.next_version[e] != before) bt.vers.push_back({(int64_t)e, B.next_version[e] - before});
      }
    }""","""        if (B.next_version[e] != before) bt.vers.push_back({(int64_t)e, B.next_version[e] - before});
      }
    }
    maya::hp_acc[10]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-tph).count();""")
g=rep(g,"""  std::vector<Chunk> chunks = device_chunks(M, (int)p, (int)v, (int)stage);""","""  auto tpro = std::chrono::steady_clock::now();
  maya::hp_acc[13]+=std::chrono::duration<double>(tpro-tstart).count();
  std::vector<Chunk> chunks = device_chunks(M, (int)p, (int)v, (int)stage);""")
g=rep(g,"""  const int64_t t = C.t, d = C.d;
  const int64_t i = rank % t""","""  auto tstart = std::chrono::steady_clock::now();
  const int64_t t = C.t, d = C.d;
  const int64_t i = rank % t""")
g=rep(g,"""  for (const Step &st : pipeline_order(schedule, p, m, v, stage)) {
    if (!tpl_on) {""","""  auto tpo = std::chrono::steady_clock::now();
  const std::vector<Step> steps_po = pipeline_order(schedule, p, m, v, stage);
  maya::hp_acc[14]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-tpo).count();
  for (const Step &st : steps_po) {
    if (!tpl_on) {""")
g=rep(g,"""  // gradient reduction and optimizer step (:757-777)""","""  auto tepi = std::chrono::steady_clock::now();
  struct EpiT { std::chrono::steady_clock::time_point t; ~EpiT(){ maya::hp_acc[15]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-t).count(); } } epit{tepi};
  // gradient reduction and optimizer step (:757-777)""")
g=rep(g,"""  const bool tpl_on = B.blocks && jtpl;""","""  maya::hp_acc[12]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-tpro).count();
  const bool tpl_on = B.blocks && jtpl;""")
open('/tmp/hprof/gen.cpp','w').write(g)
p=open('/tmp/hprof/pack.cpp').read()
p=rep(p,'#include "pack.h"','#include "pack.h"\n'+hdr+'namespace maya { double hp_acc[16]; }\n')
p=rep(p,"""  void finish() {""","""  void finish() {
    HP(3);""")
p=rep(p,"""  JobHdr &H = P.hdr;
  renumber_features(P);""","""  HP(4);
  JobHdr &H = P.hdr;
  { HP(9); renumber_features(P); }""")
p=rep(p,"""  P.collapsed = collapse && build_collapsed(job, rep_comms, V);""","""  { HP(5); P.collapsed = collapse && build_collapsed(job, rep_comms, V); }""")
p=rep(p,"""  // communicators and their call slots (JobTrace.groups / .calls)""","""  auto t6 = std::chrono::steady_clock::now();
  // communicators and their call slots (JobTrace.groups / .calls)""")
p=rep(p,"""  // work accounting over ALL ranks (sim.py:183-184)""","""  maya::hp_acc[6]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-t6).count();
  auto t7 = std::chrono::steady_clock::now();
  // work accounting over ALL ranks (sim.py:183-184)""")
p=rep(p,"""  // Collectives every simulated rank of a rep meets alone""","""  maya::hp_acc[7]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-t7).count();
  auto t8 = std::chrono::steady_clock::now();
  // Collectives every simulated rank of a rep meets alone""")
p=rep(p,"""  // walkers rank-major: a scheduler warp owns whole ranks""","""  maya::hp_acc[8]+=std::chrono::duration<double>(std::chrono::steady_clock::now()-t8).count();
  // walkers rank-major: a scheduler warp owns whole ranks""")
open('/tmp/hprof/pack.cpp','w').write(p)
EOF
g++ -O2 -std=c++17 -I/root/repo/include /root/repo/tools/hostprof/${HPP:-hpp}.cpp /tmp/hprof/gen.cpp /tmp/hprof/pack.cpp -lpthread -o /tmp/hpp && /tmp/hpp $HPP_ARGS
