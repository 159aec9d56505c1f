// partition_io.cpp -- the text side of partition metrics (metrics.cpp:90-166):
// assignment files, metrics JSON and the part-graph DOT.
//
// metrics_json (metrics.cpp:124-139) is nlohmann::json's dump(2).  The json
// library is vendored by the reference (proj/vendor, not shipped), so its
// output format is restated from the library's documented behaviour:
// object keys in std::map (sorted) order, two-space indent, ": " and ",\n"
// separators, integers in decimal, doubles as the shortest round-trip digits
// placed by dtoa_impl::format_buffer (fixed notation for decimal exponents in
// (-4, 15], otherwise d.ddde+XX with at least two exponent digits; integral
// values keep a trailing ".0").  Here the digits come from std::to_chars,
// which is the true shortest form; nlohmann's Grisu2 is shortest in all but
// rare cases.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "esg_internal.h"

namespace esg {

std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  std::string out;
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0.0) return out + "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  const std::string sci(buf, r.ptr);  // d[.ddd]e[+-]XX
  const size_t epos = sci.find('e');
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (sci[i] != '.') digits += sci[i];
  const int k = (int)digits.size();
  const int n = std::atoi(sci.c_str() + epos + 1) + 1;  // value = 0.digits * 10^n
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) return out + digits + std::string(n - k, '0') + ".0";
  if (0 < n && n <= kMaxExp) return out + digits.substr(0, n) + "." + digits.substr(n);
  if (kMinExp < n && n <= 0) return out + "0." + std::string(-n, '0') + digits;
  std::string m = digits.substr(0, 1);
  if (k > 1) m += "." + digits.substr(1);
  int e = n - 1;
  char eb[16];
  std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
  return out + m + eb;
}

std::string metrics_json(const esg_metrics& m, const esg_part_stats* parts) {
  std::ostringstream o;
  o << "{\n";
  o << "  \"cut_edges\": " << m.cut_edges << ",\n";
  o << "  \"edge_imbalance\": " << json_double(m.edge_imbalance) << ",\n";
  o << "  \"max_neighbors\": " << m.max_neighbors << ",\n";
  o << "  \"mean_neighbors\": " << json_double(m.mean_neighbors) << ",\n";
  o << "  \"n_parts\": " << m.n_parts << ",\n";
  o << "  \"node_imbalance\": " << json_double(m.node_imbalance) << ",\n";
  if (m.n_parts == 0) {
    o << "  \"parts\": [],\n";
  } else {
    o << "  \"parts\": [\n";
    for (int q = 0; q < m.n_parts; ++q) {
      const esg_part_stats& s = parts[q];
      o << "    {\n";
      o << "      \"edges\": " << s.edges << ",\n";
      o << "      \"neighbors\": " << s.neighbors << ",\n";
      o << "      \"nodes\": " << s.nodes << ",\n";
      o << "      \"recv_volume\": " << s.recv_volume << "\n";
      o << "    }" << (q + 1 < m.n_parts ? ",\n" : "\n");
    }
    o << "  ],\n";
  }
  o << "  \"total_recv_volume\": " << m.total_recv << "\n";
  o << "}";
  return o.str();
}

// metrics.cpp:141-166: one node statement per part, then one edge statement
// per (from, to) pair with a positive volume, in (from, to) order
std::string partition_dot(const int64_t* vol, const esg_part_stats* parts, int P) {
  std::ostringstream o;
  o << "digraph parts {\n";
  for (int q = 0; q < P; ++q) o << "  p" << q << " [label=\"part " << q << "\\n" << parts[q].nodes << " nodes\"];\n";
  for (int f = 0; f < P; ++f)
    for (int q = 0; q < P; ++q)
      if (vol[(size_t)f * P + q] > 0) o << "  p" << f << " -> p" << q << " [label=\"" << vol[(size_t)f * P + q] << "\"];\n";
  o << "}\n";
  return o.str();
}

// metrics.cpp:90-93
void write_assignment(const std::string& path, const int32_t* part, int64_t n) {
  std::ofstream out(path);
  if (!out) data("cannot write " + path);
  for (int64_t i = 0; i < n; ++i) out << i << ' ' << part[i] << '\n';
  if (!out) data("cannot write " + path);
}

// metrics.cpp:101-116: ids must run 0, 1, 2, ...; parts non-negative;
// n_parts = max part + 1
std::vector<int32_t> read_assignment(const std::string& path, int* n_parts) {
  std::ifstream in(path);
  if (!in) data("cannot read " + path);
  std::vector<int32_t> out;
  int np = 0;
  long id = 0, part = 0, expect = 0;
  while (in >> id >> part) {
    if (id != expect) data("assignment line for node " + std::to_string(expect) + " found id " + std::to_string(id));
    if (part < 0) data("negative part id");
    out.push_back((int32_t)part);
    np = std::max(np, (int)part + 1);
    ++expect;
  }
  if (!in.eof() && in.fail()) data("malformed assignment file");
  if (out.empty()) data("empty assignment");
  *n_parts = np;
  return out;
}

}  // namespace esg
