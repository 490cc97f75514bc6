// Trace ingestion fast path: CSV -> fp64 samples in native code, with the
// reference's load_trace rules (trace.py:87-169):
//
//   * lines as str.splitlines() (\n, \r, \r\n, \v, \f, \x1c, \x1d, \x1e)     trace.py:107-108
//   * header: first line, stripped, must be "timestamp,capacity_w"            trace.py:110-114
//   * whitespace-only rows are skipped; a row is exactly 2 comma fields       trace.py:119-124
//   * timestamp: ISO-8601, trailing Z -> UTC, naive -> UTC, offset must be 0  trace.py:72-83
//   * capacity: float(), finite, >= 0 (-0.0 passes)                           trace.py:129-136
//   * step rule: delta > 0, delta % step == 0; whole-step gaps are an error
//     unless gap_fill, which repeats the previous sample (zero-order hold)    trace.py:138-161
//
// The native grammar is deliberately narrow: ASCII text, timestamps YYYY-MM-DD(T| )HH:MM:SS with
// an optional 1-6 digit fraction and an optional Z / z / +00:00 / -00:00 suffix, plain decimal
// capacities. Every file inside it yields exactly the reference's samples; anything else — any
// error, or a valid but exotic spelling (underscored numbers, week dates, other separators,
// non-ASCII line breaks) — stops with CS_E_UNSUPPORTED and the Python loader (the reference
// rules restated in trace.py) produces the outcome, including the exact exception. Host I/O
// only: nothing here touches the GPU.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include "cs_internal.h"

namespace cs {
namespace {

struct Parsed {
  std::vector<double> values;
  int64_t start_us = 0;
  int32_t status = CS_E_UNSUPPORTED;
  int32_t line = 0;
};

inline bool is_break(unsigned char c) {  // str.splitlines separators in ASCII (\r\n handled by caller)
  return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e;
}
inline bool is_str_space(unsigned char c) {  // str.isspace() in ASCII
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}
inline bool is_float_space(unsigned char c) {  // float() strips only these (Py_ISSPACE)
  return c == ' ' || (c >= 0x09 && c <= 0x0d);
}
inline bool dig(unsigned char c) { return c >= '0' && c <= '9'; }

int fail_invalid(const std::string& msg) {
  set_error(msg);
  return CS_E_INVALID;
}

struct Span {
  const char* b;
  const char* e;
  size_t size() const { return (size_t)(e - b); }
};

Span strip(Span s, bool (*sp)(unsigned char)) {
  while (s.b < s.e && sp((unsigned char)*s.b)) ++s.b;
  while (s.e > s.b && sp((unsigned char)s.e[-1])) --s.e;
  return s;
}

int num(const char* p, int n) {
  int v = 0;
  for (int i = 0; i < n; ++i) v = v * 10 + (p[i] - '0');
  return v;
}

// days since 1970-01-01 of a proleptic Gregorian date (Howard Hinnant's days_from_civil)
int64_t days_from_civil(int64_t y, unsigned m, unsigned d) {
  y -= m <= 2;
  const int64_t era = (y >= 0 ? y : y - 399) / 400;
  const unsigned yoe = (unsigned)(y - era * 400);
  const unsigned doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
  const unsigned doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + (int64_t)doe - 719468;
}

// _parse_timestamp (trace.py:72-83) for the native grammar; false = outside it or invalid
bool parse_ts(Span s, int64_t* us) {
  s = strip(s, is_str_space);
  const char* p = s.b;
  size_t n = s.size();
  if (n < 19) return false;
  if (!(dig(p[0]) && dig(p[1]) && dig(p[2]) && dig(p[3]) && p[4] == '-' && dig(p[5]) && dig(p[6]) && p[7] == '-' &&
        dig(p[8]) && dig(p[9]) && (p[10] == 'T' || p[10] == ' ') && dig(p[11]) && dig(p[12]) && p[13] == ':' &&
        dig(p[14]) && dig(p[15]) && p[16] == ':' && dig(p[17]) && dig(p[18])))
    return false;
  const int Y = num(p, 4), Mo = num(p + 5, 2), D = num(p + 8, 2), h = num(p + 11, 2), mi = num(p + 14, 2),
            se = num(p + 17, 2);
  static const int dim[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  if (Y < 1 || Mo < 1 || Mo > 12 || D < 1 || h > 23 || mi > 59 || se > 59) return false;
  const bool leap = (Y % 4 == 0 && Y % 100 != 0) || Y % 400 == 0;
  if (D > dim[Mo - 1] + (Mo == 2 && leap ? 1 : 0)) return false;
  size_t i = 19;
  int64_t frac = 0;
  if (i < n && p[i] == '.') {
    size_t k = i + 1;
    while (k < n && dig(p[k])) ++k;
    const size_t nd = k - i - 1;
    if (nd < 1 || nd > 6) return false;
    frac = num(p + i + 1, (int)nd);
    for (size_t z = nd; z < 6; ++z) frac *= 10;
    i = k;
  }
  const size_t rest = n - i;
  if (rest == 1 && (p[i] == 'Z' || p[i] == 'z')) {
    i += 1;
  } else if (rest == 6 && (p[i] == '+' || p[i] == '-') && !std::memcmp(p + i + 1, "00:00", 5)) {
    i += 6;
  } else if (rest != 0) {
    return false;
  }
  *us = ((days_from_civil(Y, (unsigned)Mo, (unsigned)D) * 86400 + h * 3600 + mi * 60 + se) * 1000000) + frac;
  return true;
}

// float() (trace.py:130) for plain decimals: [ws][+-](d+[.d*]|.d+)([eE][+-]d+)?[ws]
bool parse_cap(Span s, double* out) {
  s = strip(s, is_float_space);
  const char* p = s.b;
  const char* e = s.e;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  const char* body = p;
  size_t nd = 0;
  while (p < e && dig(*p)) ++p, ++nd;
  if (p < e && *p == '.') {
    ++p;
    while (p < e && dig(*p)) ++p, ++nd;
  }
  if (nd == 0) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* d0 = p;
    while (p < e && dig(*p)) ++p;
    if (p == d0) return false;
  }
  if (p != e) return false;
  double v = 0.0;
  const auto r = std::from_chars(body, e, v, std::chars_format::general);  // correctly rounded
  if (r.ec != std::errc() || r.ptr != e) return false;  // (overflow -> inf: out of the grammar)
  v = neg ? -v : v;
  if (!std::isfinite(v) || v < 0) return false;  // ValidationError in the reference
  *out = v;
  return true;
}

constexpr int64_t kMaxValues = int64_t(1) << 31;

void parse_text(const char* text, size_t len, int64_t step_seconds, bool gap_fill, Parsed& out) {
  out = Parsed{};
  for (size_t i = 0; i < len; ++i)
    if ((unsigned char)text[i] >= 0x80) return;  // non-ASCII: reference path (decode + unicode rules)
  const int64_t step_us = step_seconds * 1000000;
  out.values.reserve(len / 24 + 16);  // ~28-30 B per canonical row: one allocation
  const char* p = text;
  const char* end = text + len;
  int32_t line = 0;
  bool have_prev = false;
  int64_t prev = 0;
  while (p < end) {
    const char* q = p;
    while (q < end && !is_break((unsigned char)*q)) ++q;
    Span row{p, q};
    ++line;
    out.line = line;
    if (q < end) p = (q[0] == '\r' && q + 1 < end && q[1] == '\n') ? q + 2 : q + 1;
    else p = end;
    if (line == 1) {
      const Span h = strip(row, is_str_space);
      static const char kHeader[] = "timestamp,capacity_w";
      if (h.size() != sizeof(kHeader) - 1 || std::memcmp(h.b, kHeader, h.size())) return;
      continue;
    }
    if (strip(row, is_str_space).size() == 0) continue;
    const char* c = static_cast<const char*>(std::memchr(row.b, ',', row.size()));
    if (!c || std::memchr(c + 1, ',', (size_t)(row.e - c - 1))) return;
    int64_t ts;
    double cap;
    if (!parse_ts(Span{row.b, c}, &ts) || !parse_cap(Span{c + 1, row.e}, &cap)) return;
    if (have_prev) {
      const int64_t d = ts - prev;
      if (d <= 0 || d >= (int64_t(1) << 52) || d % step_us != 0) return;
      const int64_t missing = d / step_us - 1;
      if (missing > 0) {
        if (!gap_fill) return;
        if ((int64_t)out.values.size() + missing >= kMaxValues) return;
        out.values.insert(out.values.end(), (size_t)missing, out.values.back());
      }
    } else {
      out.start_us = ts;
      have_prev = true;
    }
    if ((int64_t)out.values.size() + 1 >= kMaxValues) return;
    out.values.push_back(cap);
    prev = ts;
  }
  if (line == 0 || out.values.empty()) return;  // empty file / no data rows: reference raises
  out.status = CS_OK;
  out.line = 0;
}

bool read_file(const char* path, std::string& buf) {  // one fstat + (usually) one read()
  const int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return false;
  struct stat st;
  bool ok = ::fstat(fd, &st) == 0;
  buf.clear();
  if (ok && st.st_size > 0) buf.resize((size_t)st.st_size);
  size_t got = 0;
  while (ok) {
    if (got == buf.size()) buf.resize(buf.size() + 65536);  // grew since fstat, or not a regular file
    const ssize_t r = ::read(fd, &buf[got], buf.size() - got);
    if (r < 0) ok = false;
    else if (r == 0) break;
    else got += (size_t)r;
  }
  ::close(fd);
  buf.resize(got);
  return ok;
}

int hw_threads(int32_t n_threads) {
  if (n_threads > 0) return n_threads;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

// f(i, worker): items i in [0, n) over `threads` workers pulling from a shared counter
template <typename F>
void parallel_for(int64_t n, int threads, F&& f) {
  threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n));
  if (threads == 1) {
    for (int64_t i = 0; i < n; ++i) f(i, 0);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (int64_t i; (i = next.fetch_add(1)) < n;) f(i, t);
    });
  for (auto& th : pool) th.join();
}

}  // namespace

struct TraceSet {
  std::vector<Parsed> traces;
};

}  // namespace cs

using cs::TraceSet;

extern "C" {

int cs_traces_parse_files(const char* const* paths, int32_t n, int64_t step_seconds, int32_t gap_fill,
                          int32_t n_threads, cs_traces** out) {
  if (!out || n < 0 || (n > 0 && !paths)) return cs::fail_invalid("null argument");
  if (step_seconds <= 0 || step_seconds > (int64_t(1) << 40)) return cs::fail_invalid("step_seconds must be positive");
  auto* ts = new TraceSet();
  ts->traces.resize((size_t)n);
  const int nt = cs::hw_threads(n_threads);
  std::vector<std::string> bufs((size_t)nt);  // one read buffer per worker, reused across files
  cs::parallel_for(n, nt, [&](int64_t i, int w) {
    std::string& buf = bufs[(size_t)w];
    cs::Parsed& p = ts->traces[(size_t)i];
    if (!paths[i] || !cs::read_file(paths[i], buf)) return;  // status stays UNSUPPORTED: the
                                                             // reference path raises the OSError
    cs::parse_text(buf.data(), buf.size(), step_seconds, gap_fill != 0, p);
  });
  *out = reinterpret_cast<cs_traces*>(ts);
  return CS_OK;
}

int cs_traces_parse_text(const char* text, int64_t len, int64_t step_seconds, int32_t gap_fill, cs_traces** out) {
  if (!out || len < 0 || (len > 0 && !text)) return cs::fail_invalid("null argument");
  if (step_seconds <= 0 || step_seconds > (int64_t(1) << 40)) return cs::fail_invalid("step_seconds must be positive");
  auto* ts = new TraceSet();
  ts->traces.resize(1);
  cs::parse_text(text, (size_t)len, step_seconds, gap_fill != 0, ts->traces[0]);
  *out = reinterpret_cast<cs_traces*>(ts);
  return CS_OK;
}

int cs_traces_info(const cs_traces* t, int32_t i, cs_trace_info* info) {
  if (!t || !info) return cs::fail_invalid("null argument");
  const auto& v = reinterpret_cast<const TraceSet*>(t)->traces;
  if (i < 0 || (size_t)i >= v.size()) return cs::fail_invalid("trace index out of range");
  info->n_values = (int64_t)v[i].values.size();
  info->start_unix_us = v[i].start_us;
  info->status = v[i].status;
  info->line = v[i].line;
  return CS_OK;
}

int cs_traces_copy(const cs_traces* t, int32_t i, double* out) {
  if (!t || !out) return cs::fail_invalid("null argument");
  const auto& v = reinterpret_cast<const TraceSet*>(t)->traces;
  if (i < 0 || (size_t)i >= v.size()) return cs::fail_invalid("trace index out of range");
  if (v[i].status != CS_OK) return cs::fail_invalid("trace was not parsed natively");
  std::memcpy(out, v[i].values.data(), v[i].values.size() * sizeof(double));
  return CS_OK;
}

int cs_traces_pack(const cs_traces* t, int32_t dtype, int64_t n_steps, int64_t ld, void* out, int32_t n_threads) {
  if (!t || !out) return cs::fail_invalid("null argument");
  if (dtype != CS_CAP_F32 && dtype != CS_CAP_F64) return cs::fail_invalid("dtype must be CS_CAP_F32 or CS_CAP_F64");
  if (n_steps < 1 || ld < n_steps) return cs::fail_invalid("need 1 <= n_steps <= ld");
  const auto& v = reinterpret_cast<const TraceSet*>(t)->traces;
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i].status != CS_OK) return cs::fail_invalid("trace " + std::to_string(i) + " was not parsed natively");
    if ((int64_t)v[i].values.size() != n_steps)
      return cs::fail_invalid("trace " + std::to_string(i) + " has " + std::to_string(v[i].values.size()) +
                              " samples, expected " + std::to_string(n_steps));
  }
  cs::parallel_for((int64_t)v.size(), cs::hw_threads(n_threads), [&](int64_t i, int) {
    const double* src = v[(size_t)i].values.data();
    if (dtype == CS_CAP_F64) {
      double* dst = static_cast<double*>(out) + i * ld;
      std::memcpy(dst, src, (size_t)n_steps * 8);
      std::fill(dst + n_steps, dst + ld, 0.0);
    } else {
      float* dst = static_cast<float*>(out) + i * ld;
      for (int64_t k = 0; k < n_steps; ++k) dst[k] = (float)src[k];
      std::fill(dst + n_steps, dst + ld, 0.0f);
    }
  });
  return CS_OK;
}

void cs_traces_destroy(cs_traces* t) { delete reinterpret_cast<TraceSet*>(t); }

}  // extern "C"
