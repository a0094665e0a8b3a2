// bal_host.cpp -- array-native reader of Bundle-Adjustment-in-the-Large problem
// files (the reference's io.read_bal, io.py:83-131).
//
// The reference tokenises the whole file into Python strings and builds one
// Python object per observation (minutes at 20M observations); this reads the
// file once into flat arrays ready for the device: cam_idx / pt_idx [N] int64,
// pixels [N][2], camera parameters [C][9] (angle-axis, translation, focal,
// k1, k2) and points [P][3]. Host code only: the Python side converts the
// camera parameters exactly as the reference does (io.py:121-124).
//
// Token and error rules follow io.py:38-76 and 83-119: '#' starts a comment
// to the end of the line, tokens split on Python whitespace, line numbers
// count Python line breaks (\n, \r, \r\n, \v, \f, \x1c-\x1e); integers and
// numbers parse like Python int() / float() (sign, underscores between
// digits, inf / nan; no hex); the same messages, line numbers and error
// classes (ParseError, CountMismatch, IndexError-free range checks,
// DuplicateObservation in observation order).
#include <stdint.h>
#include <stdio.h>
#include <algorithm>
#include <charconv>
#include <cstring>
#include <string>
#include <vector>

extern "C" int ssfm_internal_set_error(int code, const char* msg);

namespace {

enum { ST_OK = 0, ST_INVALID = 9, ST_PARSE = 12, ST_COUNT = 13, ST_DUPLICATE = 14 };

struct Reader {
  const char* p;
  const char* end;
  long long line = 1;          // line of the cursor
  long long last_line = 1;     // line of the file's last token (reference: items[-1][1])
  bool comment = false;

  static bool is_break(unsigned char c) { return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1e); }
  static bool is_space(unsigned char c) { return c == ' ' || c == '\t' || is_break(c) || c == 0x1f; }

  // next token [s, e) and its line; false at end of file
  bool next(const char** s, const char** e, long long* ln) {
    while (p < end) {
      const unsigned char c = (unsigned char)*p;
      if (is_break(c)) {
        if (c == '\r' && p + 1 < end && p[1] == '\n') ++p;
        ++p;
        ++line;
        comment = false;
        continue;
      }
      if (comment || is_space(c)) { ++p; continue; }
      if (c == '#') { comment = true; ++p; continue; }
      const char* t = p;
      while (p < end && !is_space((unsigned char)*p) && *p != '#') ++p;
      *s = t;
      *e = p;
      *ln = line;
      return true;
    }
    return false;
  }
};

std::string quoted(const char* s, const char* e) { return "'" + std::string(s, e) + "'"; }

// Python's rule: '_' only between two digits; returns the token without them
bool strip_underscores(const char* s, const char* e, std::string* out) {
  out->clear();
  for (const char* q = s; q < e; ++q) {
    if (*q == '_') {
      if (q == s || q + 1 == e || !isdigit((unsigned char)q[-1]) || !isdigit((unsigned char)q[1])) return false;
      continue;
    }
    out->push_back(*q);
  }
  return true;
}

bool parse_int(const char* s, const char* e, long long* v) {
  std::string t;
  if (!strip_underscores(s, e, &t) || t.empty()) return false;
  const char* a = t.data();
  const char* b = a + t.size();
  bool neg = false;
  if (*a == '+' || *a == '-') { neg = *a == '-'; ++a; }
  if (a == b) return false;
  unsigned long long u = 0;
  for (const char* q = a; q < b; ++q) {
    if (!isdigit((unsigned char)*q)) return false;
    if (u > (~0ull - 9) / 10) { u = ~0ull; continue; }   // saturate: out of every range below
    u = u * 10 + (unsigned)(*q - '0');
  }
  if (u > (unsigned long long)INT64_MAX) u = (unsigned long long)INT64_MAX;
  *v = neg ? -(long long)u : (long long)u;
  return true;
}

bool parse_float(const char* s, const char* e, double* v) {
  std::string t;
  if (!strip_underscores(s, e, &t) || t.empty()) return false;
  const char* a = t.data();
  const char* b = a + t.size();
  bool neg = false;
  if (*a == '+' || *a == '-') { neg = *a == '-'; ++a; }
  if (a == b || *a == '+' || *a == '-') return false;
  for (const char* q = a; q < b; ++q)
    if (*q == 'x' || *q == 'X' || *q == '(' || *q == 'p' || *q == 'P') return false;   // hex / nan(...)
  double x = 0.0;
  auto r = std::from_chars(a, b, x, std::chars_format::general);
  if (r.ec == std::errc::result_out_of_range) {
    // Python float() rounds to +-inf / 0 instead of failing
    x = strtod(std::string(a, b).c_str(), nullptr);
  } else if (r.ec != std::errc() || r.ptr != b) {
    return false;
  }
  *v = neg ? -x : x;
  return true;
}

struct Bal {
  long long C = 0, P = 0, N = 0;
  std::vector<int64_t> cam, pt;
  std::vector<double> pix, cams, pts;
};

int fail(int code, const std::string& msg) { return ssfm_internal_set_error(code, msg.c_str()); }
int parse_fail(long long ln, const std::string& why) { return fail(ST_PARSE, "line " + std::to_string(ln) + ": " + why); }

}  // namespace

struct ssfm_bal {
  Bal b;
};

extern "C" int ssfm_bal_read(const char* path, ssfm_bal** out, int64_t* counts) {
  if (!path || !out || !counts) return fail(ST_INVALID, "null argument");
  *out = nullptr;
  FILE* fh = fopen(path, "rb");
  if (!fh) return fail(ST_INVALID, std::string("cannot open ") + path);
  std::vector<char> buf;
  {
    fseek(fh, 0, SEEK_END);
    const long sz = ftell(fh);
    fseek(fh, 0, SEEK_SET);
    buf.resize(sz > 0 ? (size_t)sz : 0);
    const size_t got = sz > 0 ? fread(buf.data(), 1, buf.size(), fh) : 0;
    fclose(fh);
    if (got != buf.size()) return fail(ST_INVALID, std::string("short read of ") + path);
  }
  Reader rd{buf.data(), buf.data() + buf.size()};
  // line of the file's last token, for end-of-file messages only (rescans)
  auto last_line = [&]() {
    Reader pre{buf.data(), buf.data() + buf.size()};
    const char *s0, *e0;
    long long l0;
    while (pre.next(&s0, &e0, &l0)) pre.last_line = l0;
    return pre.last_line;
  };
  const char *s = nullptr, *e = nullptr;
  long long ln = 0;
  auto take = [&](const char* what) -> int {
    if (!rd.next(&s, &e, &ln)) return parse_fail(last_line(), std::string("unexpected end of file, expected ") + what);
    return ST_OK;
  };
  auto take_int = [&](const char* what, long long* v) -> int {
    int rc = take(what);
    if (rc) return rc;
    if (!parse_int(s, e, v)) return parse_fail(ln, std::string("expected integer ") + what + ", got " + quoted(s, e));
    return ST_OK;
  };
  // `what` is formatted only on failure: "<a>", or "<a> <i> <b> <k>" when b is set
  auto what_of = [](const char* a, long long i, const char* b2, int k) {
    return b2 ? std::string(a) + " " + std::to_string(i) + " " + b2 + " " + std::to_string(k) : std::string(a);
  };
  auto take_float = [&](double* v, const char* a, long long i = 0, const char* b2 = nullptr, int k = 0) -> int {
    if (!rd.next(&s, &e, &ln))
      return parse_fail(last_line(), "unexpected end of file, expected " + what_of(a, i, b2, k));
    if (!parse_float(s, e, v))
      return parse_fail(ln, "expected number " + what_of(a, i, b2, k) + ", got " + quoted(s, e));
    return ST_OK;
  };
  Bal b;
  int rc;
  if ((rc = take_int("camera count", &b.C)) || (rc = take_int("point count", &b.P)) ||
      (rc = take_int("observation count", &b.N)))
    return rc;
  const long long header_line = ln;
  if (std::min(b.C, std::min(b.P, b.N)) < 0) return parse_fail(header_line, "negative count in header");
  // a record takes >= 2 bytes per token: never reserve more than the file can hold
  const long long cap = (long long)buf.size() / 2 + 1;
  b.cam.reserve(std::min(b.N, cap));
  b.pt.reserve(std::min(b.N, cap));
  b.pix.reserve(2 * std::min(b.N, cap));
  for (long long k = 0; k < b.N; ++k) {
    long long ci, pi;
    double u, v;
    if ((rc = take_int("camera index", &ci))) return rc;
    const long long cl = ln;
    if ((rc = take_int("point index", &pi)) || (rc = take_float(&u, "pixel u")) || (rc = take_float(&v, "pixel v")))
      return rc;
    if (!(0 <= ci && ci < b.C))
      return parse_fail(cl, "camera index " + std::to_string(ci) + " out of range [0, " + std::to_string(b.C) + ")");
    if (!(0 <= pi && pi < b.P))
      return parse_fail(cl, "point index " + std::to_string(pi) + " out of range [0, " + std::to_string(b.P) + ")");
    b.cam.push_back(ci);
    b.pt.push_back(pi);
    b.pix.push_back(u);
    b.pix.push_back(v);
  }
  b.cams.reserve(9 * std::min(b.C, cap));
  for (long long i = 0; i < b.C; ++i)
    for (int k = 0; k < 9; ++k) {
      double x;
      if ((rc = take_float(&x, "camera", i, "parameter", k))) return rc;
      b.cams.push_back(x);
    }
  b.pts.reserve(3 * std::min(b.P, cap));
  for (long long j = 0; j < b.P; ++j)
    for (int k = 0; k < 3; ++k) {
      double x;
      if ((rc = take_float(&x, "point", j, "coordinate", k))) return rc;
      b.pts.push_back(x);
    }
  if (rd.next(&s, &e, &ln)) {
    long long rest = 1;
    const char *s2, *e2;
    long long l2;
    while (rd.next(&s2, &e2, &l2)) ++rest;
    return fail(ST_COUNT, "line " + std::to_string(ln) + ": " + std::to_string(rest) +
                              " trailing tokens after the last point record");
  }
  // validate_scene (scene.py:248-262): the first repeated (camera, point) in observation order
  if (b.N > 1) {
    std::vector<int64_t> order(b.N);
    for (long long k = 0; k < b.N; ++k) order[k] = k;
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
      return b.cam[x] != b.cam[y] ? b.cam[x] < b.cam[y] : b.pt[x] < b.pt[y];
    });
    long long first_dup = -1;
    for (long long m = 1; m < b.N; ++m) {
      const int64_t x = order[m - 1], y = order[m];
      if (b.cam[x] == b.cam[y] && b.pt[x] == b.pt[y] && (first_dup < 0 || y < first_dup)) first_dup = y;
    }
    if (first_dup >= 0)
      return fail(ST_DUPLICATE, "duplicate observation (" + std::to_string(b.cam[first_dup]) + ", " +
                                    std::to_string(b.pt[first_dup]) + ")");
  }
  counts[0] = b.C;
  counts[1] = b.P;
  counts[2] = b.N;
  ssfm_bal* h = new ssfm_bal;
  h->b = std::move(b);
  *out = h;
  return ST_OK;
}

extern "C" int ssfm_bal_take(ssfm_bal* h, int64_t* cam_idx, int64_t* pt_idx, double* pixels, double* cam_params,
                             double* points) {
  if (!h) return fail(ST_INVALID, "null reader");
  const Bal& b = h->b;
  if ((b.N && (!cam_idx || !pt_idx || !pixels)) || (b.C && !cam_params) || (b.P && !points))
    return fail(ST_INVALID, "null output array");
  if (b.N) {
    memcpy(cam_idx, b.cam.data(), sizeof(int64_t) * b.N);
    memcpy(pt_idx, b.pt.data(), sizeof(int64_t) * b.N);
    memcpy(pixels, b.pix.data(), sizeof(double) * 2 * b.N);
  }
  if (b.C) memcpy(cam_params, b.cams.data(), sizeof(double) * 9 * b.C);
  if (b.P) memcpy(points, b.pts.data(), sizeof(double) * 3 * b.P);
  return ST_OK;
}

extern "C" void ssfm_bal_free(ssfm_bal* h) { delete h; }
