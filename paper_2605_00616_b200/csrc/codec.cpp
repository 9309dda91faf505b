// codec.cpp -- native readers for the reference's on-disk formats (host C++).
//
// SURVEY.md §8f rows 1-2, the data formats either side of the oracle path:
//   * profile packs: canonical JSON written by save_pack (profile.py:275-296),
//     read by load_pack (profile.py:299-347) -> per-table SoA in the device
//     layout, ready for emu_tables_create;
//   * step traces: JSON lines of StepTraceRecord (profile.py:350-404) ->
//     record SoA for emu_tables_build.
// Both parse the well-formed documents the reference writes (any key order,
// any JSON whitespace, unknown keys skipped) with correctly rounded number
// parsing (std::from_chars == Python float()), so the arrays are bit-identical
// to the reference's.  Anything outside that subset -- a syntax error, a
// number where Python would coerce a string, NaN literals, duplicate keys --
// returns EMU_ERR_UNSUPPORTED and the Python mirror re-reads the document
// with the reference's own json path, which then raises the reference's exact
// PackFormatError / PackVersionError message.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/emu_abi.h"

namespace emu {
int fail(int code, const std::string& msg);
}
using emu::fail;

namespace {

struct Unsupported {
  std::string why;
};

struct Cursor {
  const char* p;
  const char* e;

  [[noreturn]] void bad(const char* why) const { throw Unsupported{why}; }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) p++;
  }
  bool peek(char c) {
    ws();
    return p < e && *p == c;
  }
  void expect(char c) {
    ws();
    if (p >= e || *p != c) bad("unexpected character");
    p++;
  }
  // A JSON string without escapes (the fast case for keys and values).
  // Escaped strings go through str_decoded().
  std::string_view str() {
    expect('"');
    const char* s = p;
    while (p < e && *p != '"') {
      if (*p == '\\' || (unsigned char)*p < 0x20) bad("escaped string");
      p++;
    }
    if (p >= e) bad("unterminated string");
    std::string_view v(s, (size_t)(p - s));
    p++;
    return v;
  }
  static int hexval(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
  }
  uint32_t hex4() {
    if (e - p < 4) bad("bad \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; k++) {
      const int h = hexval(p[k]);
      if (h < 0) bad("bad \\u escape");
      v = v * 16 + (uint32_t)h;
    }
    p += 4;
    return v;
  }
  // A JSON string with escapes decoded to UTF-8 (Python json semantics; lone
  // surrogates, which Python keeps as code points, are outside the subset).
  std::string str_decoded() {
    expect('"');
    std::string out;
    while (p < e && *p != '"') {
      const unsigned char ch = (unsigned char)*p;
      if (ch < 0x20) bad("control character in string");
      if (ch != '\\') {
        out.push_back((char)ch);
        p++;
        continue;
      }
      p++;
      if (p >= e) bad("truncated escape");
      const char x = *p++;
      switch (x) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (e - p < 6 || p[0] != '\\' || p[1] != 'u') bad("lone surrogate");
            p += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) bad("lone surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            bad("lone surrogate");
          }
          if (cp < 0x80) {
            out.push_back((char)cp);
          } else if (cp < 0x800) {
            out.push_back((char)(0xC0 | (cp >> 6)));
            out.push_back((char)(0x80 | (cp & 0x3F)));
          } else if (cp < 0x10000) {
            out.push_back((char)(0xE0 | (cp >> 12)));
            out.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back((char)(0x80 | (cp & 0x3F)));
          } else {
            out.push_back((char)(0xF0 | (cp >> 18)));
            out.push_back((char)(0x80 | ((cp >> 12) & 0x3F)));
            out.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back((char)(0x80 | (cp & 0x3F)));
          }
          break;
        }
        default:
          bad("bad escape");
      }
    }
    if (p >= e) bad("unterminated string");
    p++;
    return out;
  }
  // Validate the JSON number grammar; returns [s, p) and whether it is an integer literal.
  std::string_view number(bool* is_int) {
    ws();
    const char* s = p;
    if (p < e && *p == '-') p++;
    if (p >= e) bad("number");
    if (*p == '0') {
      p++;
    } else if (*p >= '1' && *p <= '9') {
      while (p < e && *p >= '0' && *p <= '9') p++;
    } else {
      bad("number");
    }
    *is_int = true;
    if (p < e && *p == '.') {
      *is_int = false;
      p++;
      if (p >= e || *p < '0' || *p > '9') bad("number");
      while (p < e && *p >= '0' && *p <= '9') p++;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      *is_int = false;
      p++;
      if (p < e && (*p == '+' || *p == '-')) p++;
      if (p >= e || *p < '0' || *p > '9') bad("number");
      while (p < e && *p >= '0' && *p <= '9') p++;
    }
    return std::string_view(s, (size_t)(p - s));
  }
  int64_t integer() {
    bool is_int;
    std::string_view v = number(&is_int);
    if (!is_int) bad("non-integer where an int is expected");
    int64_t x = 0;
    auto r = std::from_chars(v.data(), v.data() + v.size(), x);
    if (r.ec != std::errc() || r.ptr != v.data() + v.size()) bad("integer out of range");
    return x;
  }
  double real() {
    bool is_int;
    std::string_view v = number(&is_int);
    double x = 0;
    auto r = std::from_chars(v.data(), v.data() + v.size(), x);
    if (r.ec != std::errc() || r.ptr != v.data() + v.size()) bad("number out of range");
    return x;
  }
  // Skip any JSON value (unknown keys).
  void skip() {
    ws();
    if (p >= e) bad("truncated");
    const char c = *p;
    if (c == '"') {
      str_decoded();
    } else if (c == '{') {
      p++;
      if (peek('}')) {
        p++;
        return;
      }
      for (;;) {
        str_decoded();
        expect(':');
        skip();
        if (peek(',')) {
          p++;
          continue;
        }
        expect('}');
        return;
      }
    } else if (c == '[') {
      p++;
      if (peek(']')) {
        p++;
        return;
      }
      for (;;) {
        skip();
        if (peek(',')) {
          p++;
          continue;
        }
        expect(']');
        return;
      }
    } else if (c == 't' && e - p >= 4 && !memcmp(p, "true", 4)) {
      p += 4;
    } else if (c == 'f' && e - p >= 5 && !memcmp(p, "false", 5)) {
      p += 5;
    } else if (c == 'n' && e - p >= 4 && !memcmp(p, "null", 4)) {
      p += 4;
    } else {
      bool is_int;
      number(&is_int);
    }
  }
  // Iterate the members of an object: f(key) must consume the value.
  template <typename F>
  void object(F f) {
    expect('{');
    if (peek('}')) {
      p++;
      return;
    }
    for (;;) {
      const std::string_view k = str();
      expect(':');
      f(k);
      if (peek(',')) {
        p++;
        continue;
      }
      expect('}');
      return;
    }
  }
  template <typename F>
  void array(F f) {
    expect('[');
    if (peek(']')) {
      p++;
      return;
    }
    for (;;) {
      f();
      if (peek(',')) {
        p++;
        continue;
      }
      expect(']');
      return;
    }
  }
};

struct Table {
  std::vector<int64_t> tt, conc, cnt;
  std::vector<double> samples;
};

}  // namespace

struct emu_pack_parsed_s {
  int64_t schema_version = 0;
  int64_t num_gpu_blocks = 0;
  std::string metadata;  // the metadata object, canonical JSON (sorted keys, ":" and "," separators)
  // per table (decode, mixed, combined): SoA in (tt, conc) order
  std::vector<int32_t> tt[3], conc[3];
  std::vector<int64_t> off[3];
  std::vector<double> samples[3];
};

namespace {

void parse_table(Cursor& c, Table& t) {
  bool have_buckets = false;
  c.object([&](std::string_view k) {
    if (k != "buckets") {
      c.skip();
      return;
    }
    if (have_buckets) c.bad("duplicate key");
    have_buckets = true;
    c.array([&]() {
      bool ht = false, hc = false, hs = false;
      int64_t tt = 0, conc = 0, n = 0;
      c.object([&](std::string_view bk) {
        if (bk == "tt") {
          if (ht) c.bad("duplicate key");
          ht = true;
          tt = c.integer();
        } else if (bk == "conc") {
          if (hc) c.bad("duplicate key");
          hc = true;
          conc = c.integer();
        } else if (bk == "samples") {
          if (hs) c.bad("duplicate key");
          hs = true;
          c.array([&]() {
            t.samples.push_back(c.real());
            n++;
          });
        } else {
          c.skip();
        }
      });
      if (!ht || !hc || !hs) c.bad("bucket missing a field");
      if (tt < INT32_MIN || tt > INT32_MAX || conc < INT32_MIN || conc > INT32_MAX) c.bad("key outside int32");
      t.tt.push_back(tt);
      t.conc.push_back(conc);
      t.cnt.push_back(n);
    });
  });
  if (!have_buckets) c.bad("table without buckets");
}

// PhaseTable.from_buckets: stable sort by (tt, conc); samples keep file order.
void finish_table(const Table& t, std::vector<int32_t>& tt, std::vector<int32_t>& conc, std::vector<int64_t>& off,
                  std::vector<double>& samples) {
  const size_t B = t.tt.size();
  std::vector<int64_t> start(B + 1, 0);
  for (size_t b = 0; b < B; b++) start[b + 1] = start[b] + t.cnt[b];
  std::vector<uint32_t> ord(B);
  std::iota(ord.begin(), ord.end(), 0u);
  std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
    return t.tt[a] != t.tt[b] ? t.tt[a] < t.tt[b] : t.conc[a] < t.conc[b];
  });
  tt.resize(B);
  conc.resize(B);
  off.assign(B + 1, 0);
  samples.resize(t.samples.size());
  int64_t o = 0;
  for (size_t i = 0; i < B; i++) {
    const uint32_t b = ord[i];
    tt[i] = (int32_t)t.tt[b];
    conc[i] = (int32_t)t.conc[b];
    std::copy(t.samples.begin() + start[b], t.samples.begin() + start[b + 1], samples.begin() + o);
    o += t.cnt[b];
    off[i + 1] = o;
  }
}

std::string json_escape(const std::string& v) {
  std::string out = "\"";
  for (unsigned char ch : v) {
    if (ch == '"' || ch == '\\') {
      out.push_back('\\');
      out.push_back((char)ch);
    } else if (ch < 0x20) {
      char b[8];
      snprintf(b, sizeof b, "\\u%04x", ch);
      out += b;
    } else {
      out.push_back((char)ch);
    }
  }
  return out + "\"";
}

// metadata: {str: str} only (the reference converts other values with str()).
// Returned as a JSON object (UTF-8, keys sorted by code point) for the caller's
// json.loads.
std::string parse_metadata(Cursor& c) {
  std::vector<std::pair<std::string, std::string>> kv;
  c.expect('{');
  if (!c.peek('}')) {
    for (;;) {
      std::string k = c.str_decoded();
      c.expect(':');
      for (auto& x : kv)
        if (x.first == k) c.bad("duplicate key");
      c.ws();
      if (c.p >= c.e || *c.p != '"') c.bad("non-string metadata value");
      kv.emplace_back(std::move(k), c.str_decoded());
      if (c.peek(',')) {
        c.p++;
        continue;
      }
      break;
    }
  }
  c.expect('}');
  std::sort(kv.begin(), kv.end());
  std::string out = "{";
  for (size_t i = 0; i < kv.size(); i++) {
    if (i) out += ",";
    out += json_escape(kv[i].first) + ":" + json_escape(kv[i].second);
  }
  return out + "}";
}

// One JSONL trace record (profile.py:365-378): step, tt, conc ints; phase
// "decode" | "mixed"; latency_s a number.
struct TraceCols {
  int64_t* step;
  int32_t* tt;
  int32_t* conc;
  uint8_t* phase;
  double* lat;
};

void parse_trace_line(Cursor& c, TraceCols& o, int64_t i) {
  bool hs = false, ht = false, hc = false, hp = false, hl = false;
  c.object([&](std::string_view k) {
    if (k == "step") {
      if (hs) c.bad("duplicate key");
      hs = true;
      o.step[i] = c.integer();
    } else if (k == "tt") {
      if (ht) c.bad("duplicate key");
      ht = true;
      const int64_t v = c.integer();
      if (v < INT32_MIN || v > INT32_MAX) c.bad("tt outside int32");
      o.tt[i] = (int32_t)v;
    } else if (k == "conc") {
      if (hc) c.bad("duplicate key");
      hc = true;
      const int64_t v = c.integer();
      if (v < INT32_MIN || v > INT32_MAX) c.bad("conc outside int32");
      o.conc[i] = (int32_t)v;
    } else if (k == "phase") {
      if (hp) c.bad("duplicate key");
      hp = true;
      const std::string_view v = c.str();
      if (v == "decode")
        o.phase[i] = 0;
      else if (v == "mixed")
        o.phase[i] = 1;
      else
        c.bad("unknown phase");
    } else if (k == "latency_s") {
      if (hl) c.bad("duplicate key");
      hl = true;
      o.lat[i] = c.real();
    } else {
      c.skip();
    }
  });
  if (!(hs && ht && hc && hp && hl)) c.bad("record missing a field");
}

bool blank_line(const char* s, const char* e) {
  for (; s < e; s++)
    if (!(*s == ' ' || *s == '\t' || *s == '\r' || *s == '\n' || *s == '\f' || *s == '\v')) return false;
  return true;
}

}  // namespace

extern "C" {

int emu_pack_parse_json(const char* text, int64_t len, emu_pack_parsed_t* out) {
  if (!text || !out || len < 0) return fail(EMU_ERR_INVALID, "NULL text/out");
  *out = nullptr;
  auto P = std::make_unique<emu_pack_parsed_s>();
  try {
    Cursor c{text, text + len};
    bool hv = false, hm = false, hb = false, ht = false;
    Table tabs[3];
    c.object([&](std::string_view k) {
      if (k == "schema_version") {
        if (hv) c.bad("duplicate key");
        hv = true;
        P->schema_version = c.integer();
      } else if (k == "metadata") {
        if (hm) c.bad("duplicate key");
        hm = true;
        P->metadata = parse_metadata(c);
      } else if (k == "num_gpu_blocks") {
        if (hb) c.bad("duplicate key");
        hb = true;
        P->num_gpu_blocks = c.integer();
      } else if (k == "tables") {
        if (ht) c.bad("duplicate key");
        ht = true;
        bool seen[3] = {false, false, false};
        c.object([&](std::string_view tk) {
          const int id = tk == "decode" ? 0 : tk == "mixed" ? 1 : tk == "combined" ? 2 : -1;
          if (id < 0) {
            c.skip();
            return;
          }
          if (seen[id]) c.bad("duplicate key");
          seen[id] = true;
          parse_table(c, tabs[id]);
        });
        if (!(seen[0] && seen[1] && seen[2])) c.bad("missing table");
      } else {
        c.skip();
      }
    });
    c.ws();
    if (c.p != c.e) c.bad("trailing data");
    if (!hv || !hb || !ht) c.bad("missing top-level field");
    if (P->schema_version != 1) c.bad("schema version");  // PackVersionError text comes from Python
    if (!hm) P->metadata = "{}";
    for (int i = 0; i < 3; i++) finish_table(tabs[i], P->tt[i], P->conc[i], P->off[i], P->samples[i]);
  } catch (const Unsupported& u) {
    return fail(EMU_ERR_UNSUPPORTED, "pack JSON outside the native subset: " + u.why);
  } catch (const std::bad_alloc&) {
    return fail(EMU_ERR_INVALID, "out of host memory parsing the pack");
  }
  *out = P.release();
  return EMU_OK;
}

int emu_pack_parsed_info(emu_pack_parsed_t p, int64_t* schema_version, int64_t* num_gpu_blocks, int64_t* sizes,
                         int64_t* metadata_len) {
  if (!p) return fail(EMU_ERR_INVALID, "NULL parsed pack");
  if (schema_version) *schema_version = p->schema_version;
  if (num_gpu_blocks) *num_gpu_blocks = p->num_gpu_blocks;
  if (sizes)
    for (int i = 0; i < 3; i++) {
      sizes[2 * i] = (int64_t)p->tt[i].size();
      sizes[2 * i + 1] = (int64_t)p->samples[i].size();
    }
  if (metadata_len) *metadata_len = (int64_t)p->metadata.size();
  return EMU_OK;
}

int emu_pack_parsed_copy(emu_pack_parsed_t p, int table, int32_t* tt, int32_t* conc, int64_t* off, double* samples) {
  if (!p || table < 0 || table > 2) return fail(EMU_ERR_INVALID, "bad parsed pack / table id");
  const size_t B = p->tt[table].size(), N = p->samples[table].size();
  if (B && (!tt || !conc)) return fail(EMU_ERR_INVALID, "NULL key output");
  if (!off || (N && !samples)) return fail(EMU_ERR_INVALID, "NULL off/samples output");
  if (B) {
    memcpy(tt, p->tt[table].data(), 4 * B);
    memcpy(conc, p->conc[table].data(), 4 * B);
  }
  memcpy(off, p->off[table].data(), 8 * (B + 1));
  if (N) memcpy(samples, p->samples[table].data(), 8 * N);
  return EMU_OK;
}

int emu_pack_parsed_metadata(emu_pack_parsed_t p, char* buf, int64_t cap) {
  if (!p || !buf || cap < (int64_t)p->metadata.size()) return fail(EMU_ERR_INVALID, "metadata buffer too small");
  memcpy(buf, p->metadata.data(), p->metadata.size());
  return EMU_OK;
}

void emu_pack_parsed_free(emu_pack_parsed_t p) { delete p; }

int64_t emu_trace_count_lines(const char* text, int64_t len) {
  if (!text || len <= 0) return 0;
  int64_t n = 0;
  const char* p = text;
  const char* e = text + len;
  while (p < e) {
    const char* nl = (const char*)memchr(p, '\n', (size_t)(e - p));
    const char* le = nl ? nl : e;
    if (!blank_line(p, le)) n++;
    p = nl ? nl + 1 : e;
  }
  return n;
}

int emu_trace_parse_jsonl(const char* text, int64_t len, int n_threads, int64_t cap, int64_t* step, int32_t* tt,
                          int32_t* conc, uint8_t* phase, double* lat, int64_t* n_out, int64_t* bad_line) {
  if (!text || len < 0 || !n_out) return fail(EMU_ERR_INVALID, "NULL text/n_out");
  if (bad_line) *bad_line = -1;
  // Split into chunks at line boundaries; count records per chunk, then
  // parse each chunk into its slice (records keep file order).
  const int T = std::max(1, std::min(n_threads > 0 ? n_threads : 1, 64));
  std::vector<const char*> cut(T + 1);
  cut[0] = text;
  cut[T] = text + len;
  for (int k = 1; k < T; k++) {
    const char* q = text + (len * k) / T;
    if (q < cut[k - 1]) q = cut[k - 1];
    const char* nl = (const char*)memchr(q, '\n', (size_t)(text + len - q));
    cut[k] = nl ? nl + 1 : text + len;
  }
  std::vector<int64_t> cnt(T, 0), base(T + 1, 0);
  std::vector<std::thread> th;
  for (int k = 0; k < T; k++)
    th.emplace_back([&, k]() { cnt[k] = emu_trace_count_lines(cut[k], (int64_t)(cut[k + 1] - cut[k])); });
  for (auto& t : th) t.join();
  th.clear();
  for (int k = 0; k < T; k++) base[k + 1] = base[k] + cnt[k];
  *n_out = base[T];
  if (base[T] > cap) return fail(EMU_ERR_CAPACITY, "trace has more records than the output capacity");
  if (base[T] && (!step || !tt || !conc || !phase || !lat)) return fail(EMU_ERR_INVALID, "NULL output column");
  std::vector<int64_t> err(T, -1);
  TraceCols cols{step, tt, conc, phase, lat};
  for (int k = 0; k < T; k++)
    th.emplace_back([&, k]() {
      int64_t i = base[k];
      const char* p = cut[k];
      const char* e = cut[k + 1];
      while (p < e) {
        const char* nl = (const char*)memchr(p, '\n', (size_t)(e - p));
        const char* le = nl ? nl : e;
        if (!blank_line(p, le)) {
          try {
            Cursor c{p, le};
            parse_trace_line(c, cols, i);
            c.ws();
            if (c.p != c.e) c.bad("trailing data");
          } catch (const Unsupported&) {
            err[k] = i;
            return;
          }
          i++;
        }
        p = nl ? nl + 1 : e;
      }
    });
  for (auto& t : th) t.join();
  for (int k = 0; k < T; k++)
    if (err[k] >= 0) {
      if (bad_line) *bad_line = err[k];
      return fail(EMU_ERR_UNSUPPORTED, "trace record " + std::to_string(err[k]) + " outside the native subset");
    }
  return EMU_OK;
}

}  // extern "C"
