// mps_reader.h -- free-format MPS reader for large instances (SURVEY.md 8(f)
// row 4: on-device ingest), host side.
//
// Semantics are those of the reference's parse_mps (core/src/mps.cpp:
// 336-407, Parser :63-330): sections NAME / OBJSENSE / ROWS / COLUMNS / RHS
// / RANGES / BOUNDS / ENDATA; the objective row's entries dropped; columns
// numbered by first appearance, integral when first seen inside an
// INTORG/INTEND marker block; values with from_chars (an optional leading
// '+'); sides built per row type with RANGES; bounds LO UP FX FR MI PL BV UI
// LI applied in order; |v| >= infinity_threshold -> +-inf; the same error
// messages ("mps parse error at line N: ...").  The matrix itself is the
// triplet list in file order, turned into CSR by pg_csr_from_triplets on the
// device (csr_from_triplets' stable order and duplicate sums).
//
// What differs is how: the file is read into memory once; one sequential
// pass finds the section headers; the COLUMNS section -- nearly all of the
// file -- is split at line boundaries over host threads that tokenize, look
// row names up in a read-only hash map and parse values concurrently; each
// chunk keeps its own first-appearance list of column names, and the chunks'
// lists are merged in file order, so column numbering and integrality are
// exactly the sequential parser's.  The first error in file order wins, as
// in the reference.
#pragma once

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

namespace pgmps {

struct Error {
  int64_t offset;  // byte offset of the offending line (line number computed on demand)
  std::string message;
};

struct Problem {
  std::string name;
  int32_t m = 0, n = 0;
  std::vector<int32_t> rows, cols;  // triplets in file order
  std::vector<double> vals;
  std::vector<double> lhs, rhs, lower, upper;
  std::vector<uint8_t> integral;
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// whitespace tokens of one line (at most `cap`, count in *nt)
inline int tokenize(std::string_view line, std::string_view* tok, int cap) {
  int nt = 0;
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_space(line[i])) ++i;
    const size_t s = i;
    while (i < line.size() && !is_space(line[i])) ++i;
    if (i > s) {
      if (nt == cap) return cap + 1;  // more than we hold: the caller decides
      tok[nt++] = line.substr(s, i - s);
    }
  }
  return nt;
}

// parse_value (mps.cpp:55-66): locale-independent, optional leading '+'
inline bool parse_value(std::string_view t, double& v) {
  std::string_view d = t;
  if (!d.empty() && d.front() == '+') d.remove_prefix(1);
  v = 0.0;
  const auto r = std::from_chars(d.data(), d.data() + d.size(), v);
  return r.ec == std::errc{} && r.ptr == d.data() + d.size();
}

inline double norm(double v, double thr) {  // normalize_infinite (model.hpp:147-151)
  const double inf = std::numeric_limits<double>::infinity();
  return v >= thr ? inf : (v <= -thr ? -inf : v);
}

enum RowType : uint8_t { kObj, kLE, kGE, kEQ };

struct Reader {
  const char* buf;
  int64_t size;
  double thr;
  int threads;
  Problem out;
  // rows
  std::vector<RowType> row_type;  // ROWS order, objective included
  std::unordered_map<std::string_view, int32_t> row_pos;
  int32_t obj_row = -1;
  // columns
  std::unordered_map<std::string_view, int32_t> col_idx;
  std::vector<std::string_view> col_names;
  bool in_int = false;
  // sides
  std::vector<double> rhs_v, rng_v;
  std::vector<uint8_t> rhs_g, rng_g;
  bool rows_ready = false;
  struct Bound {
    std::string_view type;
    int32_t col;
    double value;
    bool has_value;
    int64_t off;
  };
  std::vector<Bound> bounds;

  [[noreturn]] void fail(int64_t off, const std::string& msg) { throw Error{off, msg}; }

  void ensure_rows() {
    if (rows_ready) return;
    out.m = (int32_t)row_type.size() - (obj_row >= 0 ? 1 : 0);
    rhs_v.assign(out.m, 0.0);
    rng_v.assign(out.m, 0.0);
    rhs_g.assign(out.m, 0);
    rng_g.assign(out.m, 0);
    rows_ready = true;
  }

  // constraint index of a row name; -1 for the objective, -2 unknown
  int32_t constraint_of(std::string_view nm) const {
    const auto it = row_pos.find(nm);
    if (it == row_pos.end()) return -2;
    const int32_t pos = it->second;
    if (row_type[pos] == kObj) return -1;
    return pos - (obj_row >= 0 && pos > obj_row ? 1 : 0);
  }

  void handle_rows(const std::string_view* t, int nt, int64_t off) {
    if (nt != 2) fail(off, "ROWS line must be '<type> <name>'");
    const char c = (char)std::toupper((unsigned char)t[0][0]);
    if (t[0].size() != 1 || (c != 'N' && c != 'L' && c != 'G' && c != 'E'))
      fail(off, "unknown row type '" + std::string(t[0]) + "'");
    if (row_pos.count(t[1])) fail(off, "duplicate row name '" + std::string(t[1]) + "'");
    const RowType rt = c == 'N' ? kObj : c == 'L' ? kLE : c == 'G' ? kGE : kEQ;
    if (rt == kObj) {
      if (obj_row >= 0) fail(off, "more than one objective (N) row");
      obj_row = (int32_t)row_type.size();
    }
    row_pos.emplace(t[1], (int32_t)row_type.size());
    row_type.push_back(rt);
  }

  int32_t column_index(std::string_view nm) {  // sequential sections (BOUNDS)
    const auto it = col_idx.find(nm);
    if (it != col_idx.end()) return it->second;
    const int32_t k = (int32_t)col_names.size();
    col_idx.emplace(nm, k);
    col_names.push_back(nm);
    out.integral.push_back(in_int ? 1 : 0);
    return k;
  }

  void handle_sides(const std::string_view* t, int nt, int64_t off, std::vector<double>& v,
                    std::vector<uint8_t>& g, const char* what) {
    if (nt < 3 || nt % 2 == 0) fail(off, std::string(what) + " line must be '<set> (<row> <value>)+'");
    for (int i = 1; i + 1 < nt; i += 2) {
      const int32_t c = constraint_of(t[i]);
      if (c == -2) fail(off, "unknown row '" + std::string(t[i]) + "'");
      double x;
      if (!parse_value(t[i + 1], x)) fail(off, "cannot parse numeric value '" + std::string(t[i + 1]) + "'");
      if (c == -1) continue;
      v[c] = x;
      g[c] = 1;
    }
  }

  void handle_bounds(const std::string_view* t, int nt, int64_t off) {
    if (nt < 3) fail(off, "BOUNDS line must be '<type> <set> <col> [value]'");
    std::string up(t[0]);
    for (char& ch : up) ch = (char)std::toupper((unsigned char)ch);
    const bool no_value = up == "FR" || up == "MI" || up == "PL" || up == "BV";
    if (!no_value && nt < 4) fail(off, "bound type " + up + " requires a value");
    Bound b;
    b.col = column_index(t[2]);
    b.has_value = nt >= 4;
    b.value = 0.0;
    if (b.has_value && !parse_value(t[3], b.value))
      fail(off, "cannot parse numeric value '" + std::string(t[3]) + "'");
    b.type = t[0];
    b.off = off;
    bounds.push_back(b);
  }

  // ---- COLUMNS, in parallel -------------------------------------------------------
  struct Chunk {
    int64_t begin = 0, end = 0;
    std::vector<std::string_view> names;       // first appearances in this chunk, in order
    std::vector<uint8_t> name_int;             // integrality at that first appearance
    std::unordered_map<std::string_view, int32_t> local;
    std::vector<int32_t> rows, cols;           // cols: local ids until remapped
    std::vector<double> vals;
    bool has_marker = false, int_at_end = false;  // block state after the chunk's last marker
    bool err = false;
    Error error;
  };

  // parse [c.begin, c.end) with the integer-block state `in_block` at its start
  void parse_columns_chunk(Chunk& c, bool in_block) {
    std::string_view tok[64];
    int64_t p = c.begin;
    while (p < c.end) {
      const char* nl = (const char*)std::memchr(buf + p, '\n', (size_t)(c.end - p));
      const int64_t e = nl ? (int64_t)(nl - buf) : c.end;
      const std::string_view line(buf + p, (size_t)(e - p));
      const int64_t off = p;
      p = e + 1;
      if (line.empty() || line[0] == '*') continue;
      int nt = tokenize(line, tok, 64);
      if (nt == 0) continue;
      std::vector<std::string_view> big;
      const std::string_view* t = tok;
      if (nt > 64) {  // a very long line: tokenize into a heap vector
        big.resize((size_t)line.size() / 2 + 2);
        nt = tokenize(line, big.data(), (int)big.size());
        t = big.data();
      }
      if (std::find(t, t + nt, std::string_view("'MARKER'")) != t + nt) {
        if (std::find(t, t + nt, std::string_view("'INTORG'")) != t + nt) in_block = true;
        else if (std::find(t, t + nt, std::string_view("'INTEND'")) != t + nt) in_block = false;
        else return chunk_fail(c, off, "marker line without INTORG/INTEND");
        c.has_marker = true;
        c.int_at_end = in_block;
        continue;
      }
      if (nt < 3 || nt % 2 == 0)
        return chunk_fail(c, off, "COLUMNS line must be '<col> (<row> <value>)+'");
      int32_t lc;
      const auto it = c.local.find(t[0]);
      if (it != c.local.end()) {
        lc = it->second;
      } else {
        lc = (int32_t)c.names.size();
        c.local.emplace(t[0], lc);
        c.names.push_back(t[0]);
        c.name_int.push_back(in_block ? 1 : 0);
      }
      for (int i = 1; i + 1 < nt; i += 2) {
        const int32_t r = constraint_of(t[i]);
        if (r == -2) return chunk_fail(c, off, "unknown row '" + std::string(t[i]) + "'");
        double v;
        if (!parse_value(t[i + 1], v))
          return chunk_fail(c, off, "cannot parse numeric value '" + std::string(t[i + 1]) + "'");
        if (r == -1) continue;  // objective coefficients are dropped
        c.rows.push_back(r);
        c.cols.push_back(lc);
        c.vals.push_back(v);
      }
    }
  }
  void chunk_fail(Chunk& c, int64_t off, const std::string& msg) {
    c.err = true;
    c.error = Error{off, msg};
  }

  void parse_columns(int64_t begin, int64_t end) {
    ensure_rows();
    const int64_t bytes = end - begin;
    int nchunk = std::max(1, std::min<int>(threads, (int)(bytes / (1 << 20)) + 1));
    std::vector<Chunk> ch(nchunk);
    // chunk boundaries at line starts
    int64_t b = begin;
    for (int k = 0; k < nchunk; ++k) {
      int64_t e = k + 1 == nchunk ? end : begin + bytes * (k + 1) / nchunk;
      if (e < b) e = b;
      if (e < end) {
        const char* nl = (const char*)std::memchr(buf + e, '\n', (size_t)(end - e));
        e = nl ? std::min<int64_t>(end, (int64_t)(nl - buf) + 1) : end;
      }
      ch[k].begin = b;
      ch[k].end = e;
      b = e;
    }
    // the integer-block state at each chunk start depends on earlier markers:
    // a quick marker scan per chunk first (markers are rare), then the parse
    std::vector<int8_t> last_marker(nchunk, -1);  // -1 none, 0 INTEND, 1 INTORG
    auto scan = [&](int k) {
      // candidate lines contain the text 'MARKER'; the decision uses the
      // same exact token tests as the parse
      const std::string_view s(buf + ch[k].begin, (size_t)(ch[k].end - ch[k].begin));
      std::vector<std::string_view> tk;
      size_t q = 0;
      while ((q = s.find("'MARKER'", q)) != std::string_view::npos) {
        const size_t nlb = s.rfind('\n', q);
        const size_t ls = nlb == std::string_view::npos ? 0 : nlb + 1;
        size_t le = s.find('\n', q);
        if (le == std::string_view::npos) le = s.size();
        const std::string_view line = s.substr(ls, le - ls);
        if (!line.empty() && line[0] != '*') {
          tk.resize(line.size() / 2 + 2);
          const int nt = tokenize(line, tk.data(), (int)tk.size());
          const auto has = [&](const char* w) {
            return std::find(tk.data(), tk.data() + nt, std::string_view(w)) != tk.data() + nt;
          };
          if (has("'MARKER'")) {
            if (has("'INTORG'")) last_marker[k] = 1;
            else if (has("'INTEND'")) last_marker[k] = 0;
          }
        }
        q = le;
      }
    };
    run_parallel(nchunk, scan);
    std::vector<uint8_t> start_state(nchunk);
    bool st = in_int;
    for (int k = 0; k < nchunk; ++k) {
      start_state[k] = st;
      if (last_marker[k] >= 0) st = last_marker[k] == 1;
    }
    static const bool timing = std::getenv("PG_MPS_TIMING") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    run_parallel(nchunk, [&](int k) { parse_columns_chunk(ch[k], start_state[k] != 0); });
    auto t1 = std::chrono::steady_clock::now();
    if (timing)
      std::fprintf(stderr, "[mps] COLUMNS %.1f MB in %d chunks: %.3f s\n", bytes / 1e6, nchunk,
                   std::chrono::duration<double>(t1 - t0).count());
    // the first error in file order (chunks are in file order)
    for (int k = 0; k < nchunk; ++k)
      if (ch[k].err) throw ch[k].error;
    in_int = st;
    // global column numbers: first appearances merged in file order
    std::vector<std::vector<int32_t>> remap(nchunk);
    for (int k = 0; k < nchunk; ++k) {
      remap[k].resize(ch[k].names.size());
      for (size_t i = 0; i < ch[k].names.size(); ++i) {
        const auto it = col_idx.find(ch[k].names[i]);
        if (it != col_idx.end()) {
          remap[k][i] = it->second;
        } else {
          const int32_t g = (int32_t)col_names.size();
          col_idx.emplace(ch[k].names[i], g);
          col_names.push_back(ch[k].names[i]);
          out.integral.push_back(ch[k].name_int[i]);
          remap[k][i] = g;
        }
      }
    }
    // triplets in file order
    std::vector<size_t> base(nchunk + 1, out.rows.size());
    for (int k = 0; k < nchunk; ++k) base[k + 1] = base[k] + ch[k].rows.size();
    out.rows.resize(base[nchunk]);
    out.cols.resize(base[nchunk]);
    out.vals.resize(base[nchunk]);
    run_parallel(nchunk, [&](int k) {
      const size_t o = base[k];
      for (size_t i = 0; i < ch[k].rows.size(); ++i) {
        out.rows[o + i] = ch[k].rows[i];
        out.cols[o + i] = remap[k][ch[k].cols[i]];
        out.vals[o + i] = ch[k].vals[i];
      }
    });
  }

  template <class F>
  void run_parallel(int n, F&& f) {
    if (n == 1) {
      f(0);
      return;
    }
    std::vector<std::thread> th;
    for (int k = 1; k < n; ++k) th.emplace_back([&, k] { f(k); });
    f(0);
    for (auto& x : th) x.join();
  }

  void run() {
    enum Sec { None, Name, ObjSense, Rows, Columns, Rhs, Ranges, Bounds } sec = None;
    bool endata = false;
    std::string_view tok[64];
    int64_t p = 0;
    while (p < size) {
      const char* nl = (const char*)std::memchr(buf + p, '\n', (size_t)(size - p));
      const int64_t e = nl ? (int64_t)(nl - buf) : size;
      std::string_view line(buf + p, (size_t)(e - p));
      const int64_t off = p;
      p = e + 1;
      if (line.empty() || line[0] == '*') continue;
      const bool header = !is_space(line[0]);
      if (sec == Columns && !header) {
        // the section's data lines up to the next header: in parallel
        int64_t q = off;
        while (q < size) {
          const char* n2 = (const char*)std::memchr(buf + q, '\n', (size_t)(size - q));
          const int64_t e2 = n2 ? (int64_t)(n2 - buf) : size;
          if (e2 > q && buf[q] != '*' && !is_space(buf[q])) break;  // next header
          q = e2 + 1;
        }
        q = std::min(q, size);
        parse_columns(off, q);
        p = q;
        continue;
      }
      int nt = tokenize(line, tok, 64);
      std::vector<std::string_view> big;
      const std::string_view* t = tok;
      if (nt > 64) {
        big.resize(line.size() / 2 + 2);
        nt = tokenize(line, big.data(), (int)big.size());
        t = big.data();
      }
      if (nt == 0) continue;
      if (header) {
        const std::string_view kw = t[0];
        if (kw == "NAME") {
          sec = Name;
          if (nt > 1) out.name = std::string(t[1]);
        } else if (kw == "OBJSENSE") {
          sec = ObjSense;
        } else if (kw == "ROWS") {
          sec = Rows;
        } else if (kw == "COLUMNS") {
          sec = Columns;
          ensure_rows();
        } else if (kw == "RHS") {
          sec = Rhs;
          ensure_rows();
        } else if (kw == "RANGES") {
          sec = Ranges;
          ensure_rows();
        } else if (kw == "BOUNDS") {
          sec = Bounds;
          ensure_rows();
        } else if (kw == "ENDATA") {
          endata = true;
          break;
        } else {
          fail(off, "unknown section '" + std::string(kw) + "'");
        }
        continue;
      }
      switch (sec) {
        case Rows: handle_rows(t, nt, off); break;
        case Rhs: handle_sides(t, nt, off, rhs_v, rhs_g, "RHS"); break;
        case Ranges: handle_sides(t, nt, off, rng_v, rng_g, "RANGES"); break;
        case Bounds: handle_bounds(t, nt, off); break;
        case None: fail(off, "data before any section header");
        default: break;  // NAME / OBJSENSE values are ignored
      }
    }
    if (!endata) throw Error{-1, "missing ENDATA"};  // the line count (getline's last line)
    auto f0 = std::chrono::steady_clock::now();
    finish();
    if (std::getenv("PG_MPS_TIMING"))
      std::fprintf(stderr, "[mps] finish %.3f s\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - f0).count());
  }

  // finish (mps.cpp:232-330): sides by row type, RANGES, bounds in order
  void finish() {
    ensure_rows();
    const double inf = std::numeric_limits<double>::infinity();
    const int32_t m = out.m;
    out.n = (int32_t)col_names.size();
    out.lhs.assign(m, -inf);
    out.rhs.assign(m, inf);
    int32_t cons = 0;
    for (size_t pos = 0; pos < row_type.size(); ++pos) {
      const RowType rt = row_type[pos];
      if (rt == kObj) continue;
      const double side = rhs_g[cons] ? norm(rhs_v[cons], thr) : 0.0;
      if (rt == kLE) out.rhs[cons] = side;
      else if (rt == kGE) out.lhs[cons] = side;
      else out.lhs[cons] = out.rhs[cons] = side;
      if (rng_g[cons]) {
        const double r = rng_v[cons];
        if (rt == kLE) out.lhs[cons] = out.rhs[cons] - std::fabs(r);
        else if (rt == kGE) out.rhs[cons] = out.lhs[cons] + std::fabs(r);
        else if (r >= 0) out.rhs[cons] = out.lhs[cons] + r;
        else out.lhs[cons] = out.rhs[cons] + r;
        out.lhs[cons] = norm(out.lhs[cons], thr);
        out.rhs[cons] = norm(out.rhs[cons], thr);
      }
      ++cons;
    }
    out.lower.assign(out.n, 0.0);
    out.upper.assign(out.n, inf);
    for (const Bound& b : bounds) {
      std::string ty(b.type);
      for (char& ch : ty) ch = (char)std::toupper((unsigned char)ch);
      double& lo = out.lower[b.col];
      double& up = out.upper[b.col];
      const double v = norm(b.value, thr);
      if (ty == "LO") lo = v;
      else if (ty == "UP") up = v;
      else if (ty == "FX") lo = up = v;
      else if (ty == "FR") { lo = -inf; up = inf; }
      else if (ty == "MI") lo = -inf;
      else if (ty == "PL") up = inf;
      else if (ty == "BV") { out.integral[b.col] = 1; lo = 0; up = 1; }
      else if (ty == "UI") { out.integral[b.col] = 1; up = v; }
      else if (ty == "LI") { out.integral[b.col] = 1; lo = v; }
      else throw Error{b.off, "unknown bound type '" + ty + "'"};
    }
  }
};

// 1-based line number of a byte offset (error messages); off < 0: the
// number of lines (the reference's line counter after the last getline)
inline int64_t line_of(const char* buf, int64_t size, int64_t off) {
  int64_t line = 1;
  const int64_t lim = off < 0 ? size : std::min(off, size);
  for (int64_t i = 0; i < lim; ++i) line += buf[i] == '\n';
  if (off < 0) line -= (size == 0 || buf[size - 1] == '\n') ? 1 : 0;
  return line;
}

}  // namespace pgmps
