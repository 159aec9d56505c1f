// extxyz_io.cpp -- extended-xyz structure files (the
// input side; the reference's format: include/esgnn/structures/extxyz.h:11-20).
//
//   line 1   atom count
//   line 2   key=value pairs, values optionally double-quoted; Lattice (nine
//            numbers, lattice vectors row by row) implies pbc "T T T", pbc
//            (three flags) overrides it; other keys are ignored
//   line 3+  "Symbol x y z [more columns ignored]", one per atom
//
// The whole file is read into memory and scanned once: a line cursor over the
// buffer, numbers by std::from_chars (correctly rounded, locale-free, like
// the reference's std::stod), no per-line stream objects -- a 192k-atom C4
// file parses in a few milliseconds.  Malformed input raises ESG_ERR_DATA
// with the line number, as the reference's ParseError (core/error.h:27-35).
// The writer prints every number with 17 significant digits (%.17g), so a
// write / read round trip is exact and the text matches the reference's
// write_extxyz byte for byte.
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <string_view>
#include <vector>

#include "esg_internal.h"

namespace esg {
namespace {

[[noreturn]] void bad(const std::string& what, long line) {
  data(what + " (line " + std::to_string(line) + ")");
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// next whitespace-delimited word of v at or after *at ("" at the end)
std::string_view word(std::string_view v, size_t* at) {
  size_t i = *at;
  while (i < v.size() && is_space(v[i])) ++i;
  size_t j = i;
  while (j < v.size() && !is_space(v[j])) ++j;
  *at = j;
  return v.substr(i, j - i);
}

double number(std::string_view w, long line) {
  double x = 0.0;
  const char* b = w.data();
  const char* e = b + w.size();
  if (!w.empty() && *b == '+') ++b;  // std::stod accepts a leading '+', from_chars does not
  const auto r = std::from_chars(b, e, x);
  if (w.empty() || r.ec != std::errc() || r.ptr != e) bad("not a number: '" + std::string(w) + "'", line);
  return x;
}

// the lines of a text buffer, numbered from 1
struct Lines {
  std::string_view text;
  size_t at = 0;
  long no = 0;
  bool next(std::string_view* line) {
    if (at >= text.size()) return false;
    const size_t nl = text.find('\n', at);
    const size_t end = nl == std::string_view::npos ? text.size() : nl;
    *line = text.substr(at, end - at);
    at = end + 1;
    ++no;
    return true;
  }
};

struct Structure {
  std::vector<double> pos;
  std::vector<int32_t> species;
  double cell[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // AtomicStructure's default (structure.h): identity
  uint8_t pbc[3] = {0, 0, 0};
};

// key=value pairs of the comment line; a value is a bare word or "a quoted
// run" (no escapes).  Only Lattice and pbc are interpreted.
void comment_line(std::string_view v, long line, Structure& s) {
  bool have_lattice = false, have_pbc = false;
  std::string_view lattice, pbc;
  size_t i = 0;
  while (i < v.size()) {
    while (i < v.size() && is_space(v[i])) ++i;
    if (i >= v.size()) break;
    const size_t k0 = i;
    while (i < v.size() && v[i] != '=' && !is_space(v[i])) ++i;
    const std::string_view key = v.substr(k0, i - k0);
    std::string_view val;
    if (i < v.size() && v[i] == '=') {
      ++i;
      if (i < v.size() && v[i] == '"') {
        const size_t close = v.find('"', i + 1);
        if (close == std::string_view::npos) bad("unterminated quote in comment line", line);
        val = v.substr(i + 1, close - i - 1);
        i = close + 1;
      } else {
        const size_t v0 = i;
        while (i < v.size() && !is_space(v[i])) ++i;
        val = v.substr(v0, i - v0);
      }
    }
    if (key == "Lattice") {
      have_lattice = true;
      lattice = val;
    } else if (key == "pbc") {
      have_pbc = true;
      pbc = val;
    }
  }
  if (have_lattice) {
    size_t at = 0;
    for (int q = 0; q < 9; ++q) {
      const std::string_view w = word(lattice, &at);
      if (w.empty()) bad("Lattice needs 9 numbers", line);
      s.cell[q] = number(w, line);
    }
    s.pbc[0] = s.pbc[1] = s.pbc[2] = 1;
  }
  if (have_pbc) {
    size_t at = 0;
    for (int d = 0; d < 3; ++d) {
      const std::string_view w = word(pbc, &at);
      if (w.empty()) bad("pbc needs 3 flags", line);
      if (w == "T" || w == "True" || w == "true" || w == "1")
        s.pbc[d] = 1;
      else if (w == "F" || w == "False" || w == "false" || w == "0")
        s.pbc[d] = 0;
      else
        bad("bad pbc flag '" + std::string(w) + "'", line);
    }
  }
  if (!have_lattice && (s.pbc[0] || s.pbc[1] || s.pbc[2])) bad("pbc set but no Lattice given", line);
}

Structure parse(std::string_view text) {
  Lines in{text};
  std::string_view line;
  if (!in.next(&line)) bad("empty input", 1);
  // the count: a leading integer (words after it are ignored)
  long long n = -1;
  {
    size_t at = 0;
    const std::string_view w = word(line, &at);
    size_t len = 0;
    while (len < w.size() && (w[len] == '-' || w[len] == '+' || (w[len] >= '0' && w[len] <= '9'))) ++len;
    const char* b = w.data() + (len && w[0] == '+' ? 1 : 0);
    const auto r = std::from_chars(b, w.data() + len, n);
    if (len == 0 || r.ec != std::errc() || n < 0 || n > (1LL << 31) - 1) bad("expected atom count", in.no);
  }
  Structure s;
  if (!in.next(&line)) bad("missing comment line", 2);
  comment_line(line, in.no, s);
  s.pos.resize((size_t)n * 3);
  s.species.resize((size_t)n);
  for (long long k = 0; k < n; ++k) {
    if (!in.next(&line))
      bad("expected " + std::to_string(n) + " atom lines, got " + std::to_string(k), in.no + 1);
    size_t at = 0;
    const std::string_view sym = word(line, &at);
    std::string_view xyz[3];
    for (auto& w : xyz) w = word(line, &at);
    if (sym.empty() || xyz[2].empty()) bad("expected 'Symbol x y z'", in.no);
    s.species[k] = atomic_number(std::string(sym));
    for (int d = 0; d < 3; ++d) s.pos[3 * k + d] = number(xyz[d], in.no);
  }
  return s;
}

std::string slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) data(std::string("cannot open file: ") + path);
  return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

}  // namespace
}  // namespace esg

using namespace esg;

extern "C" {

int esg_extxyz_read(const char* path, int64_t* n_atoms, double* pos, int32_t* species, double cell[9],
                    uint8_t pbc[3]) {
  try {
    if (!path || !n_atoms) usage("null path or atom count");
    const std::string text = slurp(path);
    const Structure s = parse(text);
    *n_atoms = (int64_t)s.species.size();
    if (pos) std::memcpy(pos, s.pos.data(), sizeof(double) * s.pos.size());
    if (species) std::memcpy(species, s.species.data(), sizeof(int32_t) * s.species.size());
    if (cell) std::memcpy(cell, s.cell, sizeof(s.cell));
    if (pbc) std::memcpy(pbc, s.pbc, sizeof(s.pbc));
    return ESG_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return ESG_ERR_OTHER;
  }
}

int esg_extxyz_write(const char* path, int64_t n_atoms, const double* pos, const int32_t* species,
                     const double cell[9], const uint8_t pbc[3]) {
  try {
    if (!path || (n_atoms > 0 && (!pos || !species)) || !cell || !pbc) usage("null argument");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) data(std::string("cannot open file for writing: ") + path);
    std::string out = std::to_string(n_atoms) + "\n";
    char buf[64];
    auto num = [&](double x) {
      std::snprintf(buf, sizeof(buf), "%.17g", x);
      out += buf;
    };
    if (pbc[0] || pbc[1] || pbc[2]) {
      out += "Lattice=\"";
      for (int q = 0; q < 9; ++q) {
        num(cell[q]);
        if (q < 8) out += ' ';
      }
      out += "\" pbc=\"";
      for (int d = 0; d < 3; ++d) {
        out += pbc[d] ? 'T' : 'F';
        if (d < 2) out += ' ';
      }
      out += '"';
    }
    out += '\n';
    for (int64_t k = 0; k < n_atoms; ++k) {
      out += element_symbol(species[k]);
      for (int d = 0; d < 3; ++d) {
        out += ' ';
        num(pos[3 * k + d]);
      }
      out += '\n';
    }
    const size_t wrote = std::fwrite(out.data(), 1, out.size(), f);
    const bool ok = wrote == out.size() && std::fclose(f) == 0;
    if (!ok) data(std::string("write failed: ") + path);
    return ESG_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return ESG_ERR_OTHER;
  }
}

}  // extern "C"
