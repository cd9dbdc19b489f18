// Text trace / job manifest I/O and collation, natively (traceio.h).
//
// Messages and the order in which problems are reported follow the reference
// exactly (the parity tests compare them), including Python's repr() of the
// offending strings and int() parsing of integer fields.
#include "traceio.h"

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <thread>
#include <cstring>
#include <fstream>
#include <set>
#include <unordered_set>
#include <sstream>
#include <sys/stat.h>

namespace maya {

namespace {

const char *const KIND_NAMES[13] = {
    "HostGap", "KernelLaunch", "MemAlloc", "MemFree", "Memcpy", "Memset", "EventRecord",
    "StreamWaitEvent", "EventSynchronize", "StreamSynchronize", "DeviceSynchronize",
    "CommInit", "Collective"};
const char *const COLL_KINDS[5] = {"AllReduce", "AllGather", "ReduceScatter", "Broadcast",
                                   "SendRecv"};
const char *const TOPO_NAMES[3] = {"intra_host", "inter_host", "mixed"};

// _FIELD_ORDER (trace.py:230-244): fixed keys per kind
const std::vector<std::vector<const char *>> &field_order() {
  static const std::vector<std::vector<const char *>> F = {
      {"dur"},
      {"stream", "op", "dtype", "flops", "bytes"},
      {"id", "bytes"},
      {"id"},
      {"stream", "dir", "bytes"},
      {"stream", "bytes"},
      {"stream", "event", "ver"},
      {"stream", "event", "ver"},
      {"event", "ver"},
      {"stream"},
      {},
      {"comm", "nranks", "rank"},
      {"stream", "comm", "idx", "kind", "bytes", "nranks"}};
  return F;
}

bool has_stream(int k) {
  return k == MAYA_EV_KERNEL || k == MAYA_EV_MEMCPY || k == MAYA_EV_MEMSET ||
         k == MAYA_EV_RECORD || k == MAYA_EV_WAIT || k == MAYA_EV_SSYNC ||
         k == MAYA_EV_COLLECTIVE;
}

// Python repr() of a str (ASCII control characters escaped; other bytes kept)
std::string py_repr(const std::string &s) {
  const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
  const char q = dq ? '"' : '\'';
  std::string o(1, q);
  for (unsigned char c : s) {
    if (c == '\\') o += "\\\\";
    else if (c == (unsigned char)q) { o += '\\'; o += (char)c; }
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c == '\t') o += "\\t";
    else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", c);
      o += b;
    } else {
      o += (char)c;
    }
  }
  o += q;
  return o;
}

std::string tuple_repr(const std::vector<std::string> &v) {
  std::string o = "(";
  for (size_t i = 0; i < v.size(); i++) {
    if (i) o += ", ";
    o += py_repr(v[i]);
  }
  if (v.size() == 1) o += ",";
  return o + ")";
}

template <typename T>
std::string list_repr(const std::vector<T> &v) {
  std::string o = "[";
  for (size_t i = 0; i < v.size(); i++) {
    if (i) o += ", ";
    o += std::to_string(v[i]);
  }
  return o + "]";
}

bool py_space(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

// Python int(raw) for base-10 strings: 0 ok, 1 not an integer, 2 outside int64
int py_int(const std::string &raw, int64_t &out) {
  size_t b = 0, e = raw.size();
  while (b < e && py_space((unsigned char)raw[b])) b++;
  while (e > b && py_space((unsigned char)raw[e - 1])) e--;
  bool neg = false;
  if (b < e && (raw[b] == '+' || raw[b] == '-')) neg = raw[b++] == '-';
  if (b >= e) return 1;
  unsigned __int128 v = 0;
  bool big = false, prev_digit = false;
  for (size_t i = b; i < e; i++) {
    const char c = raw[i];
    if (c == '_') {
      if (!prev_digit || i + 1 >= e || raw[i + 1] < '0' || raw[i + 1] > '9') return 1;
      prev_digit = false;
      continue;
    }
    if (c < '0' || c > '9') return 1;
    prev_digit = true;
    if (!big) {
      v = v * 10 + (unsigned)(c - '0');
      if (v > ((unsigned __int128)1 << 64)) big = true;
    }
  }
  if (big) return 2;
  if (neg) {
    if (v > ((unsigned __int128)1 << 63)) return 2;
    out = v == ((unsigned __int128)1 << 63) ? INT64_MIN : -(int64_t)v;
  } else {
    if (v > (unsigned __int128)INT64_MAX) return 2;
    out = (int64_t)v;
  }
  return 0;
}

// fast path of py_int for plain [-]digits tokens (anything else: py_int)
int py_int_sv(std::string_view r, int64_t &out) {
  size_t i = 0;
  const bool neg = !r.empty() && r[0] == '-';
  if (neg) i = 1;
  if (i >= r.size() || r.size() - i > 18) return 1;
  int64_t v = 0;
  for (; i < r.size(); i++) {
    const char c = r[i];
    if (c < '0' || c > '9') return 1;
    v = v * 10 + (c - '0');
  }
  out = neg ? -v : v;
  return 0;
}

[[noreturn]] void parse_fail(int64_t line, const std::string &msg) {
  throw TraceFail{TERR_PARSE, "line " + std::to_string(line) + ": " + msg};
}

int64_t field_int(const std::string &raw, int64_t line, const std::string &key) {
  int64_t v = 0;
  const int rc = py_int(raw, v);
  if (rc == 1) parse_fail(line, "non-integer value for " + key + ": " + py_repr(raw));
  if (rc == 2)
    throw TraceFail{TERR_RANGE, "line " + std::to_string(line) + ": value for " + key + " " +
                                    raw + " does not fit in int64"};
  return v;
}

bool comm_id_ok(const std::string &s) {   // ^[A-Za-z0-9._-]+$
  if (s.empty()) return false;
  for (unsigned char c : s)
    if (!(isalnum(c) || c == '.' || c == '_' || c == '-')) return false;
  return true;
}
bool attr_name_ok(const std::string &s) {   // ^[a-z0-9_]+$
  if (s.empty()) return false;
  for (unsigned char c : s)
    if (!((c >= 'a' && c <= 'z') || (c >= '0' && c <= '9') || c == '_')) return false;
  return true;
}

// universal newlines (files opened in text mode): \r\n and \r end a line
std::vector<std::string_view> split_lines(const char *text, size_t len) {
  std::vector<std::string_view> out;
  size_t i = 0;
  while (i < len) {
    size_t j = i;
    while (j < len && text[j] != '\n' && text[j] != '\r') j++;
    out.emplace_back(text + i, j - i);
    if (j < len && text[j] == '\r' && j + 1 < len && text[j + 1] == '\n') j++;
    i = j + 1;
  }
  return out;
}

template <typename V>
void split_sp(std::string_view line, V &out) {   // str.split(" ")
  out.clear();
  size_t i = 0;
  for (;;) {
    const size_t j = line.find(' ', i);
    if (j == std::string_view::npos) {
      out.push_back(line.substr(i));
      return;
    }
    out.push_back(line.substr(i, j - i));
    i = j + 1;
  }
}
std::vector<std::string> split_sp(const std::string &line) {
  std::vector<std::string_view> v;
  split_sp(std::string_view(line), v);
  return std::vector<std::string>(v.begin(), v.end());
}

// trace.py:406-495, one Violation per broken rule
void validate(const ParsedTrace &t) {
  struct V {
    size_t seq;
    std::string rule, msg;
  };
  std::vector<V> out;
  struct PH {
    size_t operator()(const std::pair<int64_t, int64_t> &p) const {
      return std::hash<int64_t>()(p.first * 0x9E3779B97F4A7C15ll ^ p.second);
    }
  };
  std::unordered_set<std::pair<int64_t, int64_t>, PH> recorded;
  std::unordered_map<int64_t, int64_t> next_version;
  std::map<std::string, int64_t> comm_nranks, next_call;
  std::unordered_set<int64_t> live, seen;
  auto bad = [&](size_t seq, const char *rule, const std::string &m) { out.push_back({seq, rule, m}); };
  for (size_t seq = 0; seq < t.ev.size(); seq++) {
    const TEv &e = t.ev[seq];
    if (has_stream(e.k) && e.s < 0)
      bad(seq, "bad-stream", "negative stream handle " + std::to_string(e.s));
    switch (e.k) {
      case MAYA_EV_HOSTGAP:
        if (e.i[0] < 0) bad(seq, "negative-duration", "host gap of " + std::to_string(e.i[0]) + "ns");
        break;
      case MAYA_EV_KERNEL: {
        if (e.i[0] < 0) bad(seq, "negative-flops", "flop_count " + std::to_string(e.i[0]));
        if (e.i[1] < 0) bad(seq, "negative-bytes", "bytes_moved " + std::to_string(e.i[1]));
        const std::string &dt = t.strs[e.str[1]];
        if (dt != "fp32" && dt != "fp16" && dt != "bf16")
          bad(seq, "unknown-dtype", "dtype " + py_repr(dt));
        break;
      }
      case MAYA_EV_MEMALLOC:
        if (e.i[1] <= 0)
          bad(seq, "nonpositive-bytes", "alloc of " + std::to_string(e.i[1]) + " bytes");
        if (live.count(e.i[0]))
          bad(seq, "duplicate-alloc", "alloc_id " + std::to_string(e.i[0]) + " already live");
        live.insert(e.i[0]);
        seen.insert(e.i[0]);
        break;
      case MAYA_EV_MEMFREE:
        if (!live.count(e.i[0])) {
          if (seen.count(e.i[0]))
            bad(seq, "double-free", "alloc_id " + std::to_string(e.i[0]) + " already freed");
          else
            bad(seq, "free-unallocated", "free of unallocated handle " + std::to_string(e.i[0]));
        } else {
          live.erase(e.i[0]);
        }
        break;
      case MAYA_EV_MEMCPY:
      case MAYA_EV_MEMSET:
        if (e.i[0] <= 0)
          bad(seq, "nonpositive-bytes",
              std::string(KIND_NAMES[e.k]) + " of " + std::to_string(e.i[0]) + " bytes");
        if (e.k == MAYA_EV_MEMCPY) {
          const std::string &d = t.strs[e.str[0]];
          if (d != "H2D" && d != "D2H" && d != "D2D") bad(seq, "bad-direction", "direction " + py_repr(d));
        }
        break;
      case MAYA_EV_RECORD: {
        auto it = next_version.find(e.i[0]);
        const int64_t want = it == next_version.end() ? 0 : it->second;
        if (e.i[1] != want)
          bad(seq, "event-version-order",
              "event " + std::to_string(e.i[0]) + " recorded version " + std::to_string(e.i[1]) +
                  ", expected " + std::to_string(want));
        next_version[e.i[0]] = std::max(want, e.i[1]) + 1;
        recorded.insert({e.i[0], e.i[1]});
        break;
      }
      case MAYA_EV_WAIT:
      case MAYA_EV_ESYNC:
        if (!recorded.count({e.i[0], e.i[1]}))
          bad(seq, "unrecorded-event",
              std::string(KIND_NAMES[e.k]) + " on unrecorded event (" + std::to_string(e.i[0]) +
                  ", v" + std::to_string(e.i[1]) + ")");
        break;
      case MAYA_EV_COMMINIT: {
        const std::string &c = t.strs[e.str[0]];
        const int64_t n = e.i[0], r = e.i[1];
        if (n < 1) bad(seq, "bad-nranks", "nranks " + std::to_string(n));
        if (!(0 <= r && r < std::max<int64_t>(n, 1)))
          bad(seq, "my-rank-range",
              "my_rank " + std::to_string(r) + " not in [0, " + std::to_string(n) + ")");
        if (!comm_id_ok(c)) bad(seq, "bad-comm-id", "comm_id " + py_repr(c));
        if (comm_nranks.count(c)) {
          bad(seq, "duplicate-comm-init", "comm " + c + " already initialized");
        } else {
          comm_nranks[c] = n;
          next_call[c] = 0;
        }
        break;
      }
      case MAYA_EV_COLLECTIVE: {
        const std::string &c = t.strs[e.str[0]], &kd = t.strs[e.str[1]];
        if (!comm_nranks.count(c)) {
          bad(seq, "unknown-comm", "collective on uninitialized comm " + c);
          break;
        }
        bool known = false;
        for (const char *x : COLL_KINDS) known = known || kd == x;
        if (!known) bad(seq, "bad-collective-kind", "kind " + py_repr(kd));
        if (e.i[1] <= 0)
          bad(seq, "nonpositive-bytes", "collective of " + std::to_string(e.i[1]) + " bytes");
        const int64_t want = next_call[c];
        if (e.i[0] != want)
          bad(seq, "call-idx-order",
              "comm " + c + " call_idx " + std::to_string(e.i[0]) + ", expected " +
                  std::to_string(want));
        next_call[c] = want + 1;
        if (e.i[2] != comm_nranks[c])
          bad(seq, "nranks-mismatch",
              "collective nranks " + std::to_string(e.i[2]) + " != communicator " +
                  std::to_string(comm_nranks[c]));
        break;
      }
      default:
        break;
    }
  }
  if (out.empty()) return;
  std::string head;
  for (size_t q = 0; q < out.size() && q < 5; q++) {
    if (q) head += "; ";
    head += "seq " + std::to_string(out[q].seq) + ": [" + out[q].rule + "] " + out[q].msg;
  }
  if (out.size() > 5) head += " (+" + std::to_string(out.size() - 5) + " more)";
  throw TraceFail{TERR_VALIDATION, "invalid trace: " + head};
}

int64_t field_int(std::string_view raw, int64_t line, const char *key) {
  return field_int(std::string(raw), line, std::string(key));
}

void parse_lines(const std::vector<std::string_view> &lines, ParsedTrace &t) {
  t = ParsedTrace();
  if (lines.empty()) parse_fail(1, "empty input, missing header");
  {  // ^dltsim-trace (\S+) rank=(\d+) host=(\d+) device=(\d+)\s*$
    const std::string h(lines[0]);
    size_t e = h.size();
    while (e > 0 && py_space((unsigned char)h[e - 1])) e--;
    const std::string hs = h.substr(0, e);
    size_t b0 = 0;
    while (b0 < hs.size() && py_space((unsigned char)hs[b0])) b0++;
    const std::string shown = hs.substr(b0);
    bool ok = hs.compare(0, 13, "dltsim-trace ") == 0;
    size_t p = 13;
    std::string ver;
    std::string digs[3];
    if (ok) {
      while (p < hs.size() && !py_space((unsigned char)hs[p])) ver += hs[p++];
      ok = !ver.empty();
    }
    const char *keys[3] = {" rank=", " host=", " device="};
    for (int q = 0; q < 3 && ok; q++) {
      const size_t kl = strlen(keys[q]);
      ok = hs.compare(p, kl, keys[q]) == 0;
      if (!ok) break;
      p += kl;
      while (p < hs.size() && hs[p] >= '0' && hs[p] <= '9') digs[q] += hs[p++];
      ok = !digs[q].empty();
    }
    ok = ok && p == hs.size();
    if (!ok) parse_fail(1, "bad header: " + py_repr(shown));
    if (ver != "v1") parse_fail(1, "unsupported schema version " + py_repr(ver));
    t.rank = field_int(digs[0], 1, std::string("rank"));
    t.host = field_int(digs[1], 1, std::string("host"));
    t.device = field_int(digs[2], 1, std::string("device"));
  }
  const auto &FO = field_order();
  std::vector<std::string_view> parts, keys, vals;
  std::vector<std::pair<std::string, int64_t>> dims;
  t.ev.reserve(lines.size());
  for (size_t ln = 1; ln < lines.size(); ln++) {
    const int64_t line_no = (int64_t)ln + 1;
    const std::string_view line = lines[ln];
    if (line.empty()) continue;
    split_sp(line, parts);
    if (parts.size() < 2) parse_fail(line_no, "malformed line: " + py_repr(std::string(line)));
    int64_t seq = 0;
    if (py_int_sv(parts[0], seq) != 0) seq = field_int(parts[0], line_no, "seq");
    if (seq != (int64_t)t.ev.size())
      parse_fail(line_no, "non-monotone seq: expected " + std::to_string(t.ev.size()) + ", got " +
                              std::to_string(seq));
    keys.clear();
    vals.clear();
    for (size_t q = 2; q < parts.size(); q++) {
      const size_t eq = parts[q].find('=');
      if (eq == std::string_view::npos)
        parse_fail(line_no, "malformed key=value token " + py_repr(std::string(parts[q])));
      keys.push_back(parts[q].substr(0, eq));
      vals.push_back(parts[q].substr(eq + 1));
    }
    const std::string_view kind = parts[1];
    int k = -1;
    for (int q = 0; q < 13 && k < 0; q++)
      if (kind == KIND_NAMES[q]) k = q;
    if (k < 0) parse_fail(line_no, "unknown event kind " + py_repr(std::string(kind)));
    const std::vector<const char *> &exp = FO[k];
    {
      bool same = keys.size() >= exp.size();
      for (size_t q = 0; same && q < exp.size(); q++) same = keys[q] == exp[q];
      if (!same) {
        std::vector<std::string> got, want;
        for (size_t q = 0; q < keys.size() && q < exp.size(); q++) got.emplace_back(keys[q]);
        for (const char *x : exp) want.push_back(x);
        parse_fail(line_no, std::string(kind) + " expects keys " + tuple_repr(want) + ", got " +
                                tuple_repr(got));
      }
    }
    if (k != MAYA_EV_KERNEL && keys.size() > exp.size())
      parse_fail(line_no, std::string(kind) + " takes no extra keys, got " +
                              py_repr(std::string(keys[exp.size()])));
    // field j of the kind's fixed keys
    auto I = [&](size_t j) {
      int64_t v = 0;
      if (py_int_sv(vals[j], v) != 0) v = field_int(vals[j], line_no, exp[j]);
      return v;
    };
    auto S = [&](size_t j) { return t.intern(vals[j]); };
    TEv e{};
    e.k = (uint8_t)k;
    switch (k) {
      case MAYA_EV_HOSTGAP: e.i[0] = I(0); break;
      case MAYA_EV_KERNEL: {
        dims.clear();
        for (size_t q = exp.size(); q < keys.size(); q++) {
          const std::string_view key = keys[q];
          if (key.substr(0, 2) != "a.")
            parse_fail(line_no, "kernel attr keys must start with 'a.', got " + py_repr(std::string(key)));
          const std::string name(key.substr(2));
          if (!attr_name_ok(name)) parse_fail(line_no, "bad attr name " + py_repr(name));
          int64_t v = 0;
          if (py_int_sv(vals[q], v) != 0) v = field_int(vals[q], line_no, std::string(key).c_str());
          dims.emplace_back(name, v);
        }
        if (!std::is_sorted(dims.begin(), dims.end()))
          parse_fail(line_no, "kernel attrs must be sorted by name");
        e.s = I(0);
        e.str[0] = S(1);
        e.str[1] = S(2);
        e.i[0] = I(3);
        e.i[1] = I(4);
        e.d0 = (uint32_t)t.dims.size();
        t.dims.insert(t.dims.end(), dims.begin(), dims.end());
        e.d1 = (uint32_t)t.dims.size();
        break;
      }
      case MAYA_EV_MEMALLOC: e.i[0] = I(0); e.i[1] = I(1); break;
      case MAYA_EV_MEMFREE: e.i[0] = I(0); break;
      case MAYA_EV_MEMCPY: e.s = I(0); e.str[0] = S(1); e.i[0] = I(2); break;
      case MAYA_EV_MEMSET: e.s = I(0); e.i[0] = I(1); break;
      case MAYA_EV_RECORD:
      case MAYA_EV_WAIT: e.s = I(0); e.i[0] = I(1); e.i[1] = I(2); break;
      case MAYA_EV_ESYNC: e.i[0] = I(0); e.i[1] = I(1); break;
      case MAYA_EV_SSYNC: e.s = I(0); break;
      case MAYA_EV_DSYNC: break;
      case MAYA_EV_COMMINIT: e.str[0] = S(0); e.i[0] = I(1); e.i[1] = I(2); break;
      default:   // Collective
        e.s = I(0);
        e.str[0] = S(1);
        e.i[0] = I(2);
        e.str[1] = S(3);
        e.i[1] = I(4);
        e.i[2] = I(5);
    }
    t.ev.push_back(e);
  }
  validate(t);
}

std::string read_file(const std::string &path) {
  FILE *f = fopen(path.c_str(), "rb");
  if (!f) throw TraceFail{TERR_IO, "[Errno 2] No such file or directory: " + py_repr(path)};
  std::string out;
  fseek(f, 0, SEEK_END);
  const long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  if (n > 0) {
    out.resize((size_t)n);
    out.resize(fread(&out[0], 1, (size_t)n, f));
  }
  fclose(f);
  return out;
}

std::string dirname_of(const std::string &p) {
  const size_t s = p.rfind('/');
  return s == std::string::npos ? std::string() : p.substr(0, s);
}
std::string join_path(const std::string &a, const std::string &b) {
  if (a.empty() || (!b.empty() && b[0] == '/')) return b;
  return a.back() == '/' ? a + b : a + "/" + b;
}

[[noreturn]] void coll_fail(const std::string &m) { throw TraceFail{TERR_COLLATION, m}; }

}  // namespace

uint32_t ParsedTrace::intern(std::string_view x) {
  if (x == last_str && last_id != UINT32_MAX) return last_id;
  auto it = str_id.find(std::string(x));
  uint32_t id;
  if (it != str_id.end()) {
    id = it->second;
  } else {
    id = (uint32_t)strs.size();
    strs.emplace_back(x);
    str_id.emplace(std::string(x), id);
  }
  last_str = strs[id];
  last_id = id;
  return id;
}

void parse_trace(const char *text, size_t len, ParsedTrace &out) {
  // (views into text)
  parse_lines(split_lines(text, len), out);
}

std::string serialize_trace(const ParsedTrace &t) {
  std::string o = "dltsim-trace v1 rank=" + std::to_string(t.rank) + " host=" +
                  std::to_string(t.host) + " device=" + std::to_string(t.device) + "\n";
  const auto &FO = field_order();
  for (size_t seq = 0; seq < t.ev.size(); seq++) {
    const TEv &e = t.ev[seq];
    o += std::to_string(seq);
    o += ' ';
    o += KIND_NAMES[e.k];
    std::vector<std::string> v;
    switch (e.k) {
      case MAYA_EV_HOSTGAP: v = {std::to_string(e.i[0])}; break;
      case MAYA_EV_KERNEL:
        v = {std::to_string(e.s), t.strs[e.str[0]], t.strs[e.str[1]], std::to_string(e.i[0]),
             std::to_string(e.i[1])};
        break;
      case MAYA_EV_MEMALLOC: v = {std::to_string(e.i[0]), std::to_string(e.i[1])}; break;
      case MAYA_EV_MEMFREE: v = {std::to_string(e.i[0])}; break;
      case MAYA_EV_MEMCPY: v = {std::to_string(e.s), t.strs[e.str[0]], std::to_string(e.i[0])}; break;
      case MAYA_EV_MEMSET: v = {std::to_string(e.s), std::to_string(e.i[0])}; break;
      case MAYA_EV_RECORD:
      case MAYA_EV_WAIT: v = {std::to_string(e.s), std::to_string(e.i[0]), std::to_string(e.i[1])}; break;
      case MAYA_EV_ESYNC: v = {std::to_string(e.i[0]), std::to_string(e.i[1])}; break;
      case MAYA_EV_SSYNC: v = {std::to_string(e.s)}; break;
      case MAYA_EV_DSYNC: break;
      case MAYA_EV_COMMINIT: v = {t.strs[e.str[0]], std::to_string(e.i[0]), std::to_string(e.i[1])}; break;
      default:
        v = {std::to_string(e.s), t.strs[e.str[0]], std::to_string(e.i[0]), t.strs[e.str[1]],
             std::to_string(e.i[1]), std::to_string(e.i[2])};
    }
    for (size_t q = 0; q < v.size(); q++) {
      o += ' ';
      o += FO[e.k][q];
      o += '=';
      o += v[q];
    }
    if (e.k == MAYA_EV_KERNEL)
      for (uint32_t d = e.d0; d < e.d1; d++)
        o += " a." + t.dims[d].first + "=" + std::to_string(t.dims[d].second);
    o += '\n';
  }
  return o;
}

// collate.py:256-372 on parsed traces, then rawtrace.from_reference's arrays
void load_job(const std::string &manifest_path, int64_t num_hosts, int64_t devices_per_host,
              int64_t capacity, GenJob &G, LoadedJob &L) {
  G.clear();
  L = LoadedJob();
  const std::string base = dirname_of(manifest_path);
  const std::string text = read_file(manifest_path);
  const std::vector<std::string_view> lines = split_lines(text.data(), text.size());
  auto strip = [](const std::string &s) {
    size_t b = 0, e = s.size();
    while (b < e && py_space((unsigned char)s[b])) b++;
    while (e > b && py_space((unsigned char)s[e - 1])) e--;
    return s.substr(b, e - b);
  };
  const std::string header = lines.empty() ? std::string() : strip(std::string(lines[0]));
  if (header.compare(0, 13, "dltsim-job v1") != 0) coll_fail("bad manifest header: " + py_repr(header));
  std::vector<ParsedTrace> traces;
  std::vector<std::pair<int64_t, int64_t>> dup_rep;   // manifest order
  std::map<int64_t, std::map<std::string, std::pair<std::string, int64_t>>> raw_maps;
  // Manifest lines in order; the rank traces are parsed afterwards on worker
  // threads, and the first failure in manifest order is the one reported (a
  // manifest-level error ends the scan, as it ends the reference's loop).
  std::vector<std::string> worker_files;
  TraceFail man_err{TERR_NONE, ""};
  for (size_t q = 1; q < lines.size() && man_err.kind == TERR_NONE; q++) try {
    const std::string line = strip(std::string(lines[q]));
    if (line.empty()) continue;
    const size_t sp = line.find(' ');
    const std::string kind = line.substr(0, sp);
    const std::string rest = sp == std::string::npos ? std::string() : line.substr(sp + 1);
    std::map<std::string, std::string> kv;
    for (const std::string &tok : split_sp(rest)) {
      const size_t eq = tok.find('=');
      if (eq == std::string::npos)
        coll_fail("dictionary update sequence element has length 1; 2 is required");
      kv[tok.substr(0, eq)] = tok.substr(eq + 1);
    }
    auto geti = [&](const char *k) {
      auto it = kv.find(k);
      if (it == kv.end()) coll_fail(std::string("manifest line lacks ") + k);
      int64_t v = 0;
      if (py_int(it->second, v) != 0)
        coll_fail("invalid literal for int() with base 10: " + py_repr(it->second));
      return v;
    };
    if (kind == "worker") {
      auto it = kv.find("file");
      if (it == kv.end()) coll_fail("manifest line lacks file");
      worker_files.push_back(join_path(base, it->second));   // parsed below, in parallel
    } else if (kind == "dup") {
      dup_rep.emplace_back(geti("rank"), geti("rep"));
    } else if (kind == "dupcomm") {
      const int64_t r = geti("rank"), my = geti("myrank");
      auto f = kv.find("from"), t2 = kv.find("to");
      if (f == kv.end() || t2 == kv.end()) coll_fail("manifest dupcomm line lacks from/to");
      raw_maps[r][f->second] = {t2->second, my};
    } else if (kind == "comm") {
      // derived; re-verified by collate below
    } else {
      coll_fail("unknown manifest line kind " + py_repr(kind));
    }
  } catch (const TraceFail &f) {
    man_err = f;
  }
  traces.resize(worker_files.size());
  {
    std::vector<TraceFail> errs(worker_files.size(), TraceFail{TERR_NONE, ""});
    std::atomic<size_t> next{0};
    auto work = [&] {
      for (size_t w; (w = next.fetch_add(1)) < worker_files.size();) {
        try {
          const std::string body = read_file(worker_files[w]);
          parse_trace(body.data(), body.size(), traces[w]);
        } catch (const TraceFail &f) {
          errs[w] = f;
        }
      }
    };
    const size_t nt = std::min<size_t>(worker_files.size(),
                                       std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (size_t q = 1; q < nt; q++) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    for (const TraceFail &f : errs)
      if (f.kind != TERR_NONE) throw f;
  }
  if (man_err.kind != TERR_NONE) throw man_err;
  // ---- collate (collate.py:256-372)
  std::map<int64_t, size_t> reps;   // rank -> traces index
  std::vector<int64_t> rep_order;   // insertion order
  for (size_t q = 0; q < traces.size(); q++) {
    if (reps.count(traces[q].rank)) coll_fail("duplicate representative ranks in input");
    reps[traces[q].rank] = q;
    rep_order.push_back(traces[q].rank);
  }
  std::map<int64_t, int64_t> expansion;   // dup rank -> rep (later lines win, as a dict)
  std::vector<int64_t> exp_order;
  for (auto &d : dup_rep) {
    if (!expansion.count(d.first)) exp_order.push_back(d.first);
    expansion[d.first] = d.second;
  }
  for (int64_t r : exp_order) {
    if (reps.count(r)) coll_fail("rank " + std::to_string(r) + " is both representative and duplicate");
    if (!reps.count(expansion[r]))
      coll_fail("duplicate rank " + std::to_string(r) + " references missing rep " +
                std::to_string(expansion[r]));
  }
  std::vector<int64_t> all_ranks;
  for (auto &x : reps) all_ranks.push_back(x.first);
  for (auto &x : expansion) all_ranks.push_back(x.first);
  std::sort(all_ranks.begin(), all_ranks.end());
  const int64_t ndev = num_hosts * devices_per_host;
  bool cover = (int64_t)all_ranks.size() == ndev;
  for (size_t q = 0; cover && q < all_ranks.size(); q++) cover = all_ranks[q] == (int64_t)q;
  if (!cover) {
    std::vector<int64_t> head(all_ranks.begin(), all_ranks.begin() + std::min<size_t>(4, all_ranks.size()));
    coll_fail("job covers ranks " + list_repr(head) + "..., cluster expects 0.." +
              std::to_string(ndev - 1));
  }
  for (int64_t r : rep_order) {
    const ParsedTrace &tr = traces[reps[r]];
    const int64_t ph = r / devices_per_host, pd = r % devices_per_host;
    if (tr.host != ph || tr.device != pd)
      coll_fail("rank " + std::to_string(r) + " trace claims slot (host " + std::to_string(tr.host) +
                ", device " + std::to_string(tr.device) + ") but cluster places it at (" +
                std::to_string(ph) + ", " + std::to_string(pd) + ")");
  }
  auto rep_of = [&](int64_t r) { auto it = expansion.find(r); return it == expansion.end() ? r : it->second; };
  // rep CommInits in order (comm id, nranks, my_rank)
  struct CI { std::string id; int64_t n, my; };
  std::map<int64_t, std::vector<CI>> inits;
  for (auto &x : reps) {
    const ParsedTrace &tr = traces[x.second];
    auto &v = inits[x.first];
    for (const TEv &e : tr.ev)
      if (e.k == MAYA_EV_COMMINIT) v.push_back({tr.strs[e.str[0]], e.i[0], e.i[1]});
  }
  std::map<int64_t, std::map<std::string, std::pair<std::string, int64_t>>> comm_map;
  for (int64_t r : all_ranks) {
    auto &cm = comm_map[r];
    const auto &ri = inits[rep_of(r)];
    if (expansion.count(r)) {
      const auto &src = raw_maps[r];
      for (const CI &ci : ri)
        if (!src.count(ci.id))
          coll_fail("expansion for rank " + std::to_string(r) + " lacks translation for comm " + ci.id);
      for (const CI &ci : ri) cm[ci.id] = src.at(ci.id);
    } else {
      for (const CI &ci : ri) cm[ci.id] = {ci.id, ci.my};
    }
  }
  std::map<std::string, std::map<int64_t, int64_t>> members;
  std::map<std::string, int64_t> declared;
  for (int64_t r : all_ranks)
    for (const CI &ci : inits[rep_of(r)]) {
      const auto &m = comm_map[r][ci.id];
      auto d = declared.emplace(m.first, ci.n);
      if (d.first->second != ci.n) coll_fail("comm " + m.first + ": inconsistent nranks declarations");
      auto &slot = members[m.first];
      if (slot.count(m.second))
        coll_fail("comm " + m.first + ": position " + std::to_string(m.second) + " claimed by ranks " +
                  std::to_string(slot[m.second]) + " and " + std::to_string(r));
      slot[m.second] = r;
    }
  for (auto &x : members) {
    const int64_t n = declared[x.first];
    bool ok = (int64_t)x.second.size() == n;
    int64_t q = 0;
    for (auto &p : x.second) ok = ok && p.first == q++;
    if (!ok) {
      std::vector<int64_t> missing;
      for (int64_t p = 0; p < n; p++)
        if (!x.second.count(p)) missing.push_back(p);
      coll_fail("comm " + x.first + ": unresolved positions " + list_repr(missing) + " of " +
                std::to_string(n));
    }
    CommGroupRec g{n, {}, 0};
    std::set<int64_t> hosts;
    for (int64_t p = 0; p < n; p++) {
      g.ranks.push_back(x.second[p]);
      hosts.insert(x.second[p] / devices_per_host);
    }
    g.topo = hosts.size() == 1 ? 0 : (int64_t)hosts.size() == n ? 1 : 2;
    L.groups[x.first] = g;
  }
  // per-rep call sequences by comm (first-appearance order), then per group
  struct Call { int64_t idx; std::string kind; int64_t bytes, n; };
  std::map<int64_t, std::vector<std::pair<std::string, std::vector<Call>>>> rep_calls;
  for (auto &x : reps) {
    const ParsedTrace &tr = traces[x.second];
    auto &per = rep_calls[x.first];
    std::map<std::string, size_t> pos;
    for (const TEv &e : tr.ev) {
      if (e.k != MAYA_EV_COLLECTIVE) continue;
      const std::string &c = tr.strs[e.str[0]];
      auto it = pos.find(c);
      if (it == pos.end()) {
        it = pos.emplace(c, per.size()).first;
        per.push_back({c, {}});
      }
      per[it->second].second.push_back({e.i[0], tr.strs[e.str[1]], e.i[1], e.i[2]});
    }
  }
  std::map<std::string, std::map<int64_t, const std::vector<Call> *>> seen_by;
  for (int64_t r : all_ranks)
    for (auto &pc : rep_calls[rep_of(r)]) seen_by[comm_map[r].at(pc.first).first][r] = &pc.second;
  std::map<std::pair<std::string, int64_t>, std::pair<int, int64_t>> calls;
  for (auto &x : seen_by) {
    auto git = L.groups.find(x.first);
    if (git == L.groups.end())
      coll_fail("collective on comm " + x.first + " without CommInit resolution");
    const CommGroupRec &g = git->second;
    std::vector<int64_t> absent;
    for (int64_t r : g.ranks)
      if (!x.second.count(r)) absent.push_back(r);
    if (!absent.empty())
      coll_fail("unmatched collective: comm " + x.first + " never joined by ranks " + list_repr(absent));
    const int64_t ref_rank = g.ranks[0];
    const std::vector<Call> &ref = *x.second[ref_rank];
    for (size_t q = 1; q < g.ranks.size(); q++) {
      const int64_t r = g.ranks[q];
      const std::vector<Call> &other = *x.second[r];
      if (other.size() != ref.size())
        coll_fail("unmatched collective: comm " + x.first + " idx " +
                  std::to_string(std::min(other.size(), ref.size())) + " missing on rank " +
                  std::to_string(other.size() < ref.size() ? r : ref_rank));
      for (size_t c = 0; c < ref.size(); c++) {
        const Call &a = ref[c], &b = other[c];
        if (a.idx != b.idx || a.kind != b.kind || a.bytes != b.bytes || a.n != b.n)
          coll_fail("inconsistent collective on comm " + x.first + " idx " + std::to_string(a.idx) +
                    ": rank " + std::to_string(ref_rank) + " says (" + a.kind + "," +
                    std::to_string(a.bytes) + "b,n" + std::to_string(a.n) + "), rank " +
                    std::to_string(r) + " says (" + b.kind + "," + std::to_string(b.bytes) + "b,n" +
                    std::to_string(b.n) + ")");
      }
    }
    for (const Call &c : ref) {
      if (c.n != g.nranks)
        coll_fail("comm " + x.first + " idx " + std::to_string(c.idx) + ": event nranks " +
                  std::to_string(c.n) + " != group " + std::to_string(g.nranks));
      int kd = 0;
      while (kd < 5 && c.kind != COLL_KINDS[kd]) kd++;
      calls[{x.first, c.idx}] = {kd, c.bytes};
    }
  }
  // ---- raw arrays (rawtrace.from_reference)
  G.num_ranks = (int32_t)all_ranks.size();
  G.num_hosts = (int32_t)num_hosts;
  G.devices_per_host = (int32_t)devices_per_host;
  G.capacity = capacity;
  std::map<int64_t, int32_t> rep_index;
  for (auto &x : reps) {
    rep_index[x.first] = (int32_t)G.rep_ranks.size();
    G.rep_ranks.push_back(x.first);
  }
  for (int64_t r : all_ranks) G.rank_rep.push_back(rep_index[rep_of(r)]);
  std::map<std::string, int32_t> comm_id;
  for (auto &x : L.groups) {
    comm_id[x.first] = (int32_t)G.comm_names.size();
    G.comm_names.push_back(x.first);
    G.comm_nranks.push_back((int32_t)x.second.nranks);
    G.comm_topo.push_back((int8_t)x.second.topo);
  }
  std::vector<int64_t> ncalls(G.comm_names.size(), 0);
  for (auto &c : calls) {
    if (c.first.second < 0) throw TraceFail{TERR_RANGE, "negative call_idx on " + c.first.first};
    int64_t &m = ncalls[comm_id[c.first.first]];
    m = std::max(m, c.first.second + 1);
  }
  G.call_off.assign(1, 0);
  for (int64_t n : ncalls) G.call_off.push_back(G.call_off.back() + n);
  G.call_kind.assign(G.call_off.back(), -1);
  G.call_bytes.assign(G.call_off.back(), 0);
  for (auto &c : calls) {
    const int64_t k = G.call_off[comm_id[c.first.first]] + c.first.second;
    G.call_kind[k] = (int8_t)c.second.first;
    G.call_bytes[k] = c.second.second;
  }
  std::map<std::string, int64_t> ops, dts;
  auto op_id = [&](const std::string &s) {
    auto it = ops.emplace(s, (int64_t)L.op_names.size());
    if (it.second) L.op_names.push_back(s);
    return it.first->second;
  };
  auto dt_id = [&](const std::string &s) {
    auto it = dts.emplace(s, (int64_t)L.dtype_names.size());
    if (it.second) L.dtype_names.push_back(s);
    return it.first->second;
  };
  std::map<int64_t, std::vector<std::string>> local_order;
  G.ev_off.assign(1, 0);
  for (auto &x : reps) {
    const ParsedTrace &tr = traces[x.second];
    std::map<std::string, int64_t> local;
    auto &order = local_order[x.first];
    for (const TEv &e : tr.ev)
      if (e.k == MAYA_EV_COMMINIT && local.emplace(tr.strs[e.str[0]], (int64_t)order.size()).second)
        order.push_back(tr.strs[e.str[0]]);
    for (const TEv &e : tr.ev) {
      if (e.s < INT32_MIN || e.s > INT32_MAX)
        throw TraceFail{TERR_RANGE, "stream handle " + std::to_string(e.s) + " outside int32"};
      int64_t f[4] = {0, 0, 0, 0};
      switch (e.k) {
        case MAYA_EV_HOSTGAP: f[0] = e.i[0]; break;
        case MAYA_EV_KERNEL:
          f[0] = op_id(tr.strs[e.str[0]]);
          f[1] = dt_id(tr.strs[e.str[1]]);
          f[2] = e.i[0];
          f[3] = e.i[1];
          break;
        case MAYA_EV_MEMALLOC: f[0] = e.i[0]; f[1] = e.i[1]; break;
        case MAYA_EV_MEMFREE: f[0] = e.i[0]; break;
        case MAYA_EV_MEMCPY: {
          const std::string &d = tr.strs[e.str[0]];
          f[0] = op_id(d == "H2D" ? "memcpy_h2d" : d == "D2H" ? "memcpy_d2h" : "memcpy_d2d");
          f[1] = dt_id("fp32");
          f[3] = e.i[0];
          break;
        }
        case MAYA_EV_MEMSET:
          f[0] = op_id("memset");
          f[1] = dt_id("fp32");
          f[3] = e.i[0];
          break;
        case MAYA_EV_RECORD:
        case MAYA_EV_WAIT:
        case MAYA_EV_ESYNC: f[0] = e.i[0]; f[1] = e.i[1]; break;
        case MAYA_EV_COMMINIT: f[0] = local[tr.strs[e.str[0]]]; f[1] = e.i[0]; f[2] = e.i[1]; break;
        case MAYA_EV_COLLECTIVE: {
          f[0] = local.at(tr.strs[e.str[0]]);
          f[1] = e.i[0];
          int kd = 0;
          while (kd < 5 && tr.strs[e.str[1]] != COLL_KINDS[kd]) kd++;
          f[2] = kd;
          f[3] = e.i[1];
          break;
        }
        default: break;
      }
      G.ev_kind.push_back(e.k);
      G.ev_stream.push_back((int32_t)e.s);
      G.ev_f.insert(G.ev_f.end(), f, f + 4);
    }
    G.ev_off.push_back((int64_t)G.ev_kind.size());
  }
  G.rank_comm_off.assign(1, 0);
  for (int64_t r : all_ranks) {
    for (const std::string &c : local_order[rep_of(r)]) G.rank_comm.push_back(comm_id[comm_map[r][c].first]);
    G.rank_comm_off.push_back((int64_t)G.rank_comm.size());
  }
  for (size_t q = 0; q < G.comm_names.size(); q++) {
    if (q) G.comm_blob += '\n';
    G.comm_blob += G.comm_names[q];
  }
  // what save_job writes
  L.num_ranks = (int64_t)all_ranks.size();
  for (auto &x : reps) L.reps[x.first] = std::move(traces[x.second]);
  for (auto &x : expansion) {
    L.dup_of[x.first] = x.second;
    L.dup_comm[x.first] = comm_map[x.first];
  }
}

std::string save_job(const LoadedJob &L, const std::string &out_dir,
                     const std::string &manifest_name) {
  mkdir(out_dir.c_str(), 0777);
  std::string m = "dltsim-job v1 ranks=" + std::to_string(L.num_ranks);
  for (auto &x : L.reps) {
    const std::string fname = "rank_" + std::to_string(x.first) + ".trace";
    const std::string body = serialize_trace(x.second);
    FILE *f = fopen(join_path(out_dir, fname).c_str(), "wb");
    if (!f) throw TraceFail{TERR_IO, "cannot write " + join_path(out_dir, fname)};
    fwrite(body.data(), 1, body.size(), f);
    fclose(f);
    m += "\nworker rank=" + std::to_string(x.first) + " file=" + fname;
  }
  for (auto &x : L.dup_of) {
    m += "\ndup rank=" + std::to_string(x.first) + " rep=" + std::to_string(x.second);
    for (auto &c : L.dup_comm.at(x.first))
      m += "\ndupcomm rank=" + std::to_string(x.first) + " from=" + c.first + " to=" +
           c.second.first + " myrank=" + std::to_string(c.second.second);
  }
  for (auto &x : L.groups) {
    m += "\ncomm id=" + x.first + " nranks=" + std::to_string(x.second.nranks) + " topo=" +
         TOPO_NAMES[x.second.topo] + " ranks=";
    for (size_t q = 0; q < x.second.ranks.size(); q++)
      m += (q ? "," : "") + std::to_string(x.second.ranks[q]);
  }
  m += "\n";
  const std::string path = join_path(out_dir, manifest_name);
  FILE *f = fopen(path.c_str(), "wb");
  if (!f) throw TraceFail{TERR_IO, "cannot write " + path};
  fwrite(m.data(), 1, m.size(), f);
  fclose(f);
  return path;
}

}  // namespace maya
