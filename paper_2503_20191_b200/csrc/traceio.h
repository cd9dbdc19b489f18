// Text trace and job-manifest I/O (row f3 of SURVEY §8f), natively:
//   parse_trace / serialize_trace / validate_trace   pkg/src/dltsim/trace.py:282-495
//   save_job / load_job                               pkg/src/dltsim/collate.py:377-431
//   collate (group resolution, call tables)           pkg/src/dltsim/collate.py:256-372
// A loaded job becomes the engine's raw job (GenJob arrays) directly, with the
// string tables rawtrace.from_reference would build (same interning order),
// so a rank_<r>.trace set at GB scale never becomes Python objects.
#pragma once
#include <map>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "gen.h"

namespace maya {

enum TraceErrKind { TERR_NONE = 0, TERR_PARSE = 1, TERR_VALIDATION = 2, TERR_COLLATION = 3,
                    TERR_RANGE = 4, TERR_IO = 5 };

struct TraceFail {
  int kind;
  std::string msg;
};

// One parsed worker trace, keeping everything serialize_trace writes.
struct TEv {
  uint8_t k;           // MAYA_EV_* (trace.py EVENT_KINDS order)
  int64_t s;           // stream (0 when the kind has none)
  int64_t i[3];        // integer fields in _FIELD_ORDER order (see traceio.cpp)
  uint32_t str[2];     // string fields (ids into ParsedTrace::strs)
  uint32_t d0, d1;     // kernel attr dims [d0, d1) in ParsedTrace::dims
};
struct ParsedTrace {
  int64_t rank = 0, host = 0, device = 0;
  std::vector<TEv> ev;
  std::vector<std::string> strs;
  std::unordered_map<std::string, uint32_t> str_id;
  std::vector<std::pair<std::string, int64_t>> dims;
  std::string last_str;
  uint32_t last_id = UINT32_MAX;
  uint32_t intern(std::string_view x);
};

// parse_trace (incl. validate_trace); throws TraceFail.
void parse_trace(const char *text, size_t len, ParsedTrace &out);
std::string serialize_trace(const ParsedTrace &t);

struct CommGroupRec {
  int64_t nranks;
  std::vector<int64_t> ranks;
  int topo;            // 0 intra_host, 1 inter_host, 2 mixed
};
// Everything save_job writes, kept beside the raw job of a loaded manifest.
struct LoadedJob {
  int64_t num_ranks = 0;
  std::map<int64_t, ParsedTrace> reps;
  std::map<int64_t, int64_t> dup_of;
  std::map<int64_t, std::map<std::string, std::pair<std::string, int64_t>>> dup_comm;
  std::map<std::string, CommGroupRec> groups;
  std::vector<std::string> op_names, dtype_names;
};

// load_job(manifest, cluster) -> collate -> raw arrays in G (rawtrace.from_reference
// layout); throws TraceFail.
void load_job(const std::string &manifest_path, int64_t num_hosts, int64_t devices_per_host,
              int64_t capacity, GenJob &G, LoadedJob &L);
// save_job: rank_<r>.trace per representative + the manifest; returns its path.
std::string save_job(const LoadedJob &L, const std::string &out_dir,
                     const std::string &manifest_name);

}  // namespace maya
