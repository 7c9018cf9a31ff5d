// pmh_ingest.h -- host-side ingestion of the reference CLI's "id weight"
// text (cli._read_weighted_lines, cli.py:60-70) straight into CSR arrays.
//
// Grammar accepted here (the well-formed subset of what the reference
// accepts): per line, after stripping whitespace, empty lines and lines
// starting with '#' are skipped; otherwise the first whitespace-separated
// token is the id as Python int(tok, 0) reads it -- decimal without leading
// zeros, or 0x / 0o / 0b prefixed, '_' allowed between digits, optional '+'
// -- and the optional second token the weight as Python float() reads it
// (strtod syntax plus '_' between digits, inf / nan spelled out); further
// tokens are ignored; a missing weight is 1.0.  Anything else (negative ids,
// ids >= 2^64, malformed numbers) stops the parse with the 1-based line
// number so the caller can hand that input to the exact Python restatement,
// which raises the reference's own errors.  No device code.
#pragma once
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <string>

namespace pmh_ingest {

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

inline int digit_val(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return 99;
}

// digits with Python's underscore rule (single '_' only between digits)
inline bool parse_digits(const char* s, const char* e, int base, bool allow_leading_us,
                         uint64_t* out) {
  if (s >= e) return false;
  uint64_t v = 0;
  bool prev_us = !allow_leading_us;  // '_' not allowed first unless after a prefix
  bool any = false;
  for (const char* q = s; q < e; q++) {
    if (*q == '_') {
      if (prev_us) return false;
      prev_us = true;
      continue;
    }
    const int d = digit_val(*q);
    if (d >= base) return false;
    const unsigned __int128 nv = (unsigned __int128)v * (unsigned)base + (unsigned)d;
    if (nv >> 64) return false;
    v = (uint64_t)nv;
    prev_us = false;
    any = true;
  }
  if (prev_us || !any) return false;
  *out = v;
  return true;
}

// int(tok, 0) for a non-negative id < 2^64; false if outside the grammar
inline bool parse_id(const char* s, const char* e, uint64_t* out) {
  if (s < e && *s == '+') s++;
  if (s >= e) return false;
  if (s[0] == '0' && e - s >= 2 && ((s[1] | 0x20) >= 'a' && (s[1] | 0x20) <= 'z')) {
    const char p = (char)(s[1] | 0x20);
    const int base = p == 'x' ? 16 : p == 'o' ? 8 : p == 'b' ? 2 : 0;
    if (!base) return false;
    return parse_digits(s + 2, e, base, true, out);   // int('0x_1f', 0) is valid
  }
  if (s[0] == '0') {  // base 0: a leading zero only in all-zero literals
    for (const char* q = s; q < e; q++)
      if (*q != '0' && *q != '_') return false;
  }
  return parse_digits(s, e, 10, false, out);
}

// float(tok): strtod over the token with single '_' between digits removed
inline bool parse_weight(const char* s, const char* e, double* out) {
  std::string t;
  t.reserve((size_t)(e - s));
  for (const char* q = s; q < e; q++) {
    if (*q == '_') {
      const bool ok = q > s && q + 1 < e && q[-1] >= '0' && q[-1] <= '9' && q[1] >= '0' && q[1] <= '9';
      if (!ok) return false;
      continue;
    }
    t.push_back(*q);
  }
  // Python float() does not accept hex floats or "infinity" abbreviations
  // beyond inf / infinity / nan (any case, optional sign)
  for (char c : t)
    if (c == 'x' || c == 'X' || c == 'p' || c == 'P') return false;
  char* end = nullptr;
  const double v = strtod(t.c_str(), &end);
  if (end != t.c_str() + t.size() || t.empty()) return false;
  if (std::isnan(v)) {  // strtod accepts nan(...) payloads; float() does not
    for (char c : t)
      if (c == '(') return false;
  }
  *out = v;
  return true;
}

// Parse buf[0, len) into ids/weights (capacity cap).  Returns the number of
// entries (>= 0), or -(line number) of the first line outside the grammar,
// or -(2^62) when more than cap entries are present.
inline int64_t parse_weighted_text(const char* buf, int64_t len, uint64_t* ids, double* w,
                                   int64_t cap) {
  int64_t n = 0, line = 0;
  const char* p = buf;
  const char* end = buf + len;
  while (p < end) {
    line++;
    const char* nl = (const char*)memchr(p, '\n', (size_t)(end - p));
    const char* le = nl ? nl : end;
    const char* s = p;
    while (s < le && is_ws(*s)) s++;
    const char* t = le;
    while (t > s && is_ws(t[-1])) t--;
    p = nl ? nl + 1 : end;
    if (s == t || *s == '#') continue;
    const char* a_end = s;
    while (a_end < t && !is_ws(*a_end)) a_end++;
    uint64_t id = 0;
    if (!parse_id(s, a_end, &id)) return -line;
    double wt = 1.0;
    const char* b = a_end;
    while (b < t && is_ws(*b)) b++;
    if (b < t) {
      const char* b_end = b;
      while (b_end < t && !is_ws(*b_end)) b_end++;
      if (!parse_weight(b, b_end, &wt)) return -line;
    }
    if (n >= cap) return -(int64_t(1) << 62);
    ids[n] = id;
    w[n] = wt;
    n++;
  }
  return n;
}

}  // namespace pmh_ingest
