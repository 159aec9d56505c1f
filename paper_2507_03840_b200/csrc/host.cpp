// host.cpp -- host-side C++ of the B200 path: structure prologue, Low-NN
// partitioner, comm plan, basis/head layouts, parameter registration and
// seeded init, real-basis coupling tables.  These are O(N) / O(E) integer or
// setup work that the survey keeps on the host (SURVEY.md §8(a) a1, a4, a5,
// a18); the GPU never re-derives them.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>

#include "esg_internal.h"

namespace esg {

// ------------------------------------------------------------ structures
// AtomicStructure::wrap (structure.cpp:26-38).  The fractional transform is
// inverse(cellᵀ) in adjugate form with the determinant expanded down column
// 0, and every 3-term reduction is ((a+b)+c) -- the order Eigen's fixed-size
// kernels use -- compiled without FMA contraction (see Makefile).
namespace {
inline double cof(const M3& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m[i1][j1] * m[i2][j2] - m[i1][j2] * m[i2][j1];
}
M3 adjugate_inverse(const M3& m) {
  const double c00 = cof(m, 0, 0), c10 = cof(m, 1, 0), c20 = cof(m, 2, 0);
  const double det = (c00 * m[0][0] + c10 * m[1][0]) + c20 * m[2][0];
  const double inv = 1.0 / det;
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i][j] = (j == 0 && i == 0) ? c00 * inv : cof(m, j, i) * inv;
  r[0][1] = c10 * inv;
  r[0][2] = c20 * inv;
  return r;
}
inline void matvec(const M3& m, const double* x, double* y) {
  for (int i = 0; i < 3; ++i) y[i] = (m[i][0] * x[0] + m[i][1] * x[1]) + m[i][2] * x[2];
}
}  // namespace

void wrap_positions(int n, double* pos, const M3& cell, const bool pbc[3]) {
  if (!(pbc[0] || pbc[1] || pbc[2])) return;
  M3 ct;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) ct[i][j] = cell[j][i];
  const M3 to_frac = adjugate_inverse(ct);
  for (int a = 0; a < n; ++a) {
    double f[3];
    matvec(to_frac, pos + 3 * a, f);
    for (int d = 0; d < 3; ++d) {
      if (!pbc[d]) continue;
      f[d] -= std::floor(f[d]);
      if (f[d] >= 1.0) f[d] = 0.0;
    }
    matvec(ct, f, pos + 3 * a);
  }
}

// structure.cpp:18-24
double face_spacing(const M3& c, int d) {
  const auto& a = c[(d + 1) % 3];
  const auto& b = c[(d + 2) % 3];
  const double x = a[1] * b[2] - a[2] * b[1], y = a[2] * b[0] - a[0] * b[2], z = a[0] * b[1] - a[1] * b[0];
  const double area = std::sqrt((x * x + y * y) + z * z);
  if (!(area > 0.0)) data("degenerate cell");
  auto h = [&](int r0, int r1, int r2) { return c[r0][0] * (c[r1][1] * c[r2][2] - c[r1][2] * c[r2][1]); };
  return std::abs(h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1)) / area;
}

// -------------------------------------------------------------- Low-NN
// partition/lownn.cpp:23-133: recursive coordinate bisection, first uncut
// dimension, then the smallest ceil(2 r / extent) (1 for a single periodic
// cut), ties to the highest index; split at the first minimiser of
// |2*prefix - total| over in-degree weights; parts numbered left first.
namespace {
struct RcbState {
  int n;
  const double* pos;
  const M3* cell;
  const bool* pbc;
  std::vector<long> w;
  double r_cut;
  std::vector<int>* out;
  int next = 0;
};

int choose_dim(const RcbState& st, const std::vector<int>& idx, const int cuts[3], bool root) {
  for (int d = 0; d < 3; ++d)
    if (cuts[d] == 0) return d;
  long nn[3];
  for (int d = 0; d < 3; ++d) {
    double ext;
    if (root && st.pbc[d]) {
      ext = 0.0;
      for (int j = 0; j < 3; ++j) ext += std::abs((*st.cell)[j][d]);
    } else if (idx.empty()) {
      ext = 0.0;
    } else {
      double lo = std::numeric_limits<double>::max(), hi = -lo;
      for (int i : idx) {
        lo = std::min(lo, st.pos[3 * i + d]);
        hi = std::max(hi, st.pos[3 * i + d]);
      }
      ext = hi - lo;
    }
    if (cuts[d] == 1 && st.pbc[d])
      nn[d] = 1;
    else if (ext <= 0.0)
      nn[d] = std::numeric_limits<long>::max() / 4;
    else
      nn[d] = (long)std::ceil(2.0 * st.r_cut / ext);
  }
  int best = 0;
  for (int d = 1; d < 3; ++d)
    if (nn[d] <= nn[best]) best = d;
  return best;
}

void rcb(RcbState& st, std::vector<int>& idx, int cuts[3], int level, bool root) {
  if (level == 0) {
    for (int i : idx) (*st.out)[i] = st.next;
    ++st.next;
    return;
  }
  const int dim = choose_dim(st, idx, cuts, root);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) {
    const double pa = st.pos[3 * a + dim], pb = st.pos[3 * b + dim];
    return pa != pb ? pa < pb : a < b;
  });
  const int n = (int)idx.size();
  const int need = 1 << (level - 1);
  long total = 0;
  for (int i : idx) total += st.w[i];
  long prefix = 0, best = std::numeric_limits<long>::max();
  int split = need;
  for (int p = 1; p < n; ++p) {
    prefix += st.w[idx[p - 1]];
    if (p < need || p > n - need) continue;
    const long diff = std::labs(2 * prefix - total);
    if (diff < best) {
      best = diff;
      split = p;
    }
  }
  int sub[3] = {cuts[0], cuts[1], cuts[2]};
  ++sub[dim];
  std::vector<int> left(idx.begin(), idx.begin() + split), right(idx.begin() + split, idx.end());
  rcb(st, left, sub, level - 1, false);
  rcb(st, right, sub, level - 1, false);
}
}  // namespace

std::vector<int> lownn(int n, const double* pos, const M3& cell, const bool pbc[3], const int32_t* deg,
                       int depth, double r_cut) {
  if (depth < 0) usage("partition depth must be non-negative");
  if (depth >= 31 || (1 << depth) > n)
    usage("partition depth " + std::to_string(depth) + " needs at least " + std::to_string(1L << std::min(depth, 30)) +
          " atoms, have " + std::to_string(n));
  if (!(r_cut > 0.0)) usage("cutoff must be positive");
  std::vector<int> out(n, 0);
  if (depth == 0) return out;
  RcbState st{n, pos, &cell, pbc, {}, r_cut, &out};
  st.w.assign(deg, deg + n);
  if (std::all_of(st.w.begin(), st.w.end(), [](long v) { return v == 0; })) st.w.assign(n, 1);
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  int cuts[3] = {0, 0, 0};
  rcb(st, idx, cuts, depth, true);
  return out;
}

// ------------------------------------------------------------ elements
std::string element_symbol(int z) {
  static const char* t[] = {
      "",   "H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",  "Ne", "Na", "Mg", "Al", "Si", "P",  "S",
      "Cl", "Ar", "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co", "Ni", "Cu", "Zn", "Ga", "Ge", "As",
      "Se", "Br", "Kr", "Rb", "Sr", "Y",  "Zr", "Nb", "Mo", "Tc", "Ru", "Rh", "Pd", "Ag", "Cd", "In", "Sn",
      "Sb", "Te", "I",  "Xe", "Cs", "Ba", "La", "Ce", "Pr", "Nd", "Pm", "Sm", "Eu", "Gd", "Tb", "Dy", "Ho",
      "Er", "Tm", "Yb", "Lu", "Hf", "Ta", "W",  "Re", "Os", "Ir", "Pt", "Au", "Hg", "Tl", "Pb", "Bi", "Po",
      "At", "Rn", "Fr", "Ra", "Ac", "Th", "Pa", "U",  "Np", "Pu", "Am", "Cm", "Bk", "Cf", "Es", "Fm", "Md",
      "No", "Lr"};
  if (z < 1 || z > 103) data("unknown atomic number " + std::to_string(z));
  return t[z];
}

// ------------------------------------------------------- block cache
void* BlockCache::alloc(size_t bytes) {
  if (bytes == 0) return nullptr;
  auto it = free_blocks.lower_bound(bytes);  // smallest cached block that fits
  if (it != free_blocks.end() && it->first <= bytes + bytes / 4) {
    void* p = it->second;
    live[p] = it->first;
    cached -= it->first;
    free_blocks.erase(it);
    return p;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    flush();
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      throw Error(ESG_ERR_OOM, "out of device memory (" + std::to_string(bytes) + " bytes)");
    }
  }
  live[p] = bytes;
  return p;
}

void BlockCache::release(void* p) {
  if (!p) return;
  auto it = live.find(p);
  if (it == live.end()) {
    cudaFree(p);
    return;
  }
  const size_t cap = it->second;
  live.erase(it);
  while (cached + cap > budget && !free_blocks.empty()) {  // drop the largest cached blocks first
    auto big = std::prev(free_blocks.end());
    cudaFree(big->second);
    cached -= big->first;
    free_blocks.erase(big);
  }
  if (cached + cap > budget) {
    cudaFree(p);
    return;
  }
  free_blocks.emplace(cap, p);
  cached += cap;
}

void BlockCache::flush() {
  for (auto& kv : free_blocks) cudaFree(kv.second);
  free_blocks.clear();
  cached = 0;
}

// elements.cpp:32-36
int atomic_number(const std::string& symbol) {
  for (int z = 1; z <= 103; ++z)
    if (element_symbol(z) == symbol) return z;
  data("unknown element symbol: '" + symbol + "'");
}

// ------------------------------------------------------- basis / layouts
int Basis::n_orb(int z) const {
  auto it = shells.find(z);
  if (it == shells.end()) data("no basis for element " + element_symbol(z));
  int n = 0;
  for (int l : it->second) n += 2 * l + 1;
  return n;
}
int Basis::off(int z, int sh) const {
  int o = 0;
  const auto& v = shells.at(z);
  for (int i = 0; i < sh; ++i) o += 2 * v[i] + 1;
  return o;
}
int Basis::n_slots() const {
  size_t n = 0;
  for (const auto& kv : shells) n = std::max(n, kv.second.size());
  return (int)n;
}
int Basis::slot_l(int s) const {
  int l = -1;
  for (const auto& kv : shells)
    if (s < (int)kv.second.size()) l = std::max(l, kv.second[s]);
  return l;
}

int HeadLayout::segment(int a, int b, int L) const {
  for (size_t k = 0; k < keys.size(); ++k)
    if (keys[k].sa == a && keys[k].sb == b && keys[k].L == L) return offsets[k];
  data("no head for requested slots");
}

// layout.h:79-93
HeadLayout head_layout(const Basis& b) {
  HeadLayout h;
  const int s = b.n_slots();
  for (int sa = 0; sa < s; ++sa)
    for (int sb = 0; sb < s; ++sb)
      for (int L = 0; L <= b.slot_l(sa) + b.slot_l(sb); ++L) {
        h.keys.push_back({sa, sb, L});
        h.offsets.push_back(h.out_len);
        h.out_len += 2 * L + 1;
        h.max_l = std::max(h.max_l, L);
      }
  return h;
}

// layout.h:28-45: m = 0 rows (l ascending), then per m the -m column then the
// +m column, each l = m..l_max.
MLayout m_layout(int l_max) {
  MLayout lay;
  lay.l_max = l_max;
  lay.h = (l_max + 1) * (l_max + 1);
  lay.to_m.assign(lay.h, -1);
  lay.to_l.assign(lay.h, -1);
  lay.m_offset.assign(l_max + 1, 0);
  int pos = 0;
  for (int l = 0; l <= l_max; ++l) lay.to_m[l * l + l] = pos++;
  for (int m = 1; m <= l_max; ++m) {
    lay.m_offset[m] = pos;
    for (int sign : {-1, 1})
      for (int l = m; l <= l_max; ++l) lay.to_m[l * l + l + sign * m] = pos++;
  }
  for (int i = 0; i < lay.h; ++i) lay.to_l[lay.to_m[i]] = i;
  return lay;
}

// ------------------------------------------------------------- params
void ParamSet::add(const std::string& n, int r, int c, int f) {
  if (index.count(n)) data("duplicate parameter: " + n);
  index[n] = (int)entries.size();
  entries.push_back({n, r, c, f, total});
  total += (int64_t)r * c;
}
const ParamEntry& ParamSet::at(const std::string& n) const {
  auto it = index.find(n);
  if (it == index.end()) data("unknown parameter: " + n);
  return entries[it->second];
}

// network.h:243-276: embed per species (ascending Z), radial lift, per layer
// node/edge lin1 (3E->2E) and lin2 (2E->E) per order, attention, then heads.
ParamSet register_params(const esg_model_config& cfg, const Basis& b, const HeadLayout& h) {
  ParamSet p;
  const MLayout lay = m_layout(cfg.l_max);
  const int e = cfg.e_width;
  for (const auto& kv : b.shells) p.add("embed/" + element_symbol(kv.first), 1, e, e);
  p.add("radial/lift", e, cfg.n_radial, cfg.n_radial);
  auto so2 = [&](const std::string& base, int cin, int cout) {
    p.add(base + "/m0", lay.nd(0) * cout, lay.nd(0) * cin, lay.nd(0) * cin);
    for (int m = 1; m <= cfg.l_max; ++m) {
      const int nd = lay.nd(m);
      for (const char* ri : {"r", "i"}) p.add(base + "/m" + std::to_string(m) + ri, nd * cout, nd * cin, nd * cin);
    }
  };
  for (int layer = 0; layer < cfg.layers; ++layer) {
    for (const char* blk : {"node", "edge"}) {
      const std::string base = "layer" + std::to_string(layer) + "/" + blk;
      so2(base + "/lin1", 3 * e, 2 * e);
      so2(base + "/lin2", 2 * e, e);
    }
    p.add("layer" + std::to_string(layer) + "/att", 1, e, e);
  }
  for (const char* set : {"node", "edge"})
    for (const auto& k : h.keys)
      p.add(std::string("head/") + set + "/s" + std::to_string(k.sa) + "s" + std::to_string(k.sb) + "L" +
                std::to_string(k.L),
            1, e, e);
  return p;
}

namespace {
uint64_t fnv(const void* bytes, size_t n, uint64_t h) {
  const unsigned char* q = static_cast<const unsigned char*>(bytes);
  for (size_t i = 0; i < n; ++i) h = (h ^ q[i]) * 1099511628211ull;
  return h;
}
}  // namespace

// params.h:84-92: one mt19937_64 per entry seeded by fnv1a(name, seed ^
// golden), uniform in +-sqrt(6/fan_in) drawn in double and cast to float.
void init_params(const ParamSet& p, uint64_t seed, std::vector<float>& out) {
  out.assign(p.total, 0.0f);
  for (const auto& e : p.entries) {
    std::mt19937_64 rng(fnv(e.name.data(), e.name.size(), seed ^ 0x9e3779b97f4a7c15ull));
    const double bound = std::sqrt(6.0 / e.fan_in);
    std::uniform_real_distribution<double> u(-bound, bound);
    for (int64_t k = 0; k < (int64_t)e.rows * e.cols; ++k) out[e.offset + k] = static_cast<float>(u(rng));
  }
}

// params.h:95-102
uint64_t param_hash(const ParamSet& p, const std::vector<float>& v) {
  uint64_t h = 1469598103934665603ull;
  for (const auto& e : p.entries) {
    h = fnv(e.name.data(), e.name.size(), h);
    h = fnv(v.data() + e.offset, sizeof(float) * (size_t)e.rows * e.cols, h);
  }
  return h;
}

// ------------------------------------------------------- coupling tables
// clebsch_gordan.cpp:22-140.  Complex CG vectors per L: the top state
// |L, L> is the stretched product basis vector orthogonalised (twice) against
// the |L', L> states of every larger L' and sign-fixed positive on
// (ma=la, mb=L-la); lower states follow from J- = Ja- + Jb- with a
// renormalisation at each step.  The real block is then
// B_L * cg * (B_la (x) B_lb)^H with one fixed phase (imaginary part when
// la+lb-L is odd).  Same operation order as the CPU oracle, so the tables
// agree to the bit and block export is bit-exact against it.
namespace {
using cplx = std::complex<double>;

std::vector<std::vector<double>> cg_states(int la, int lb) {
  const int da = 2 * la + 1, db = 2 * lb + 1, dim = da * db;
  const int l0 = std::abs(la - lb), l1 = la + lb;
  auto at = [&](int ma, int mb) { return (ma + la) * db + (mb + lb); };
  auto norm = [](const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
  };
  std::vector<std::vector<double>> st(l1 - l0 + 1);  // st[L-l0]: rows M+L, dim columns
  for (int L = l1; L >= l0; --L) {
    std::vector<double> v(dim, 0.0), rows((size_t)(2 * L + 1) * dim, 0.0);
    v[at(la, L - la)] = 1.0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int Lq = L + 1; Lq <= l1; ++Lq) {
        const double* w = &st[Lq - l0][(size_t)(L + Lq) * dim];
        double d = 0.0;
        for (int k = 0; k < dim; ++k) d += w[k] * v[k];
        for (int k = 0; k < dim; ++k) v[k] -= d * w[k];
      }
      const double n = norm(v);
      if (!(n > 1e-12)) data("degenerate coupling state");
      for (double& x : v) x /= n;
    }
    if (v[at(la, L - la)] < 0.0)
      for (double& x : v) x = -x;
    std::copy(v.begin(), v.end(), rows.begin() + (size_t)(2 * L) * dim);
    for (int M = L; M > -L; --M) {
      std::vector<double> lo(dim, 0.0);
      for (int ma = -la; ma <= la; ++ma)
        for (int mb = -lb; mb <= lb; ++mb) {
          const double c = v[at(ma, mb)];
          if (c == 0.0) continue;
          if (ma > -la) lo[at(ma - 1, mb)] += c * std::sqrt(la * (la + 1.0) - ma * (ma - 1.0));
          if (mb > -lb) lo[at(ma, mb - 1)] += c * std::sqrt(lb * (lb + 1.0) - mb * (mb - 1.0));
        }
      const double f = std::sqrt(L * (L + 1.0) - M * (M - 1.0));
      for (double& x : lo) x /= f;
      const double n = norm(lo);
      for (double& x : lo) x /= n;
      v.swap(lo);
      std::copy(v.begin(), v.end(), rows.begin() + (size_t)(L + M - 1) * dim);
    }
    st[L - l0] = std::move(rows);
  }
  return st;
}

// rows: real component index m+l; columns: complex m+l
std::vector<cplx> real_basis(int l) {
  const int d = 2 * l + 1;
  std::vector<cplx> b((size_t)d * d, cplx(0.0, 0.0));
  const double s = 1.0 / std::sqrt(2.0);
  b[(size_t)l * d + l] = 1.0;
  for (int m = 1; m <= l; ++m) {
    const double ph = (m % 2 == 0) ? 1.0 : -1.0;
    b[(size_t)(l + m) * d + (l - m)] = s;
    b[(size_t)(l + m) * d + (l + m)] = ph * s;
    b[(size_t)(l - m) * d + (l - m)] = cplx(0.0, s);
    b[(size_t)(l - m) * d + (l + m)] = cplx(0.0, -ph * s);
  }
  return b;
}
}  // namespace

std::vector<double> coupling_matrix(int la, int lb, int L) {
  if (L < std::abs(la - lb) || L > la + lb) data("coupled degree violates the triangle rule");
  const int da = 2 * la + 1, db = 2 * lb + 1, dL = 2 * L + 1, dim = da * db;
  const auto st = cg_states(la, lb);
  const auto Ba = real_basis(la), Bb = real_basis(lb), BL = real_basis(L);
  const std::vector<double>& cg = st[L - std::abs(la - lb)];
  // t = B_L * cg (dL x dim)
  std::vector<cplx> t((size_t)dL * dim, cplx(0.0, 0.0));
  for (int i = 0; i < dL; ++i)
    for (int k = 0; k < dL; ++k) {
      const cplx a = BL[(size_t)i * dL + k];
      if (a == cplx(0.0, 0.0)) continue;
      for (int j = 0; j < dim; ++j) t[(size_t)i * dim + j] += a * cg[(size_t)k * dim + j];
    }
  // u = t * K^H with K[(i,j),(k,m)] = Ba[i][k] Bb[j][m]
  std::vector<double> out((size_t)dL * dim);
  const bool odd = ((la + lb - L) & 1) != 0;
  for (int i = 0; i < dL; ++i)
    for (int q = 0; q < dim; ++q) {
      const int qa = q / db, qb = q % db;
      cplx acc(0.0, 0.0);
      for (int p = 0; p < dim; ++p) {
        const cplx kq = Ba[(size_t)qa * da + p / db] * Bb[(size_t)qb * db + p % db];
        acc += t[(size_t)i * dim + p] * std::conj(kq);
      }
      out[(size_t)i * dim + q] = odd ? acc.imag() : acc.real();
    }
  return out;
}

}  // namespace esg
