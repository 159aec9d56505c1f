// blocks_io.cpp -- shard reader and the text writer (see blocks_io.h).
#include "blocks_io.h"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>
#include <map>
#include <fstream>

#include "esg_internal.h"

namespace esg {

ShardHeader shard_header(uint32_t basis, uint32_t value_bytes, uint32_t flags, uint32_t rank, uint32_t world,
                         uint64_t n_blocks, uint64_t n_values) {
  ShardHeader h{};
  std::memcpy(h.magic, "ESGBLKS1", 8);
  h.version = 1;
  h.basis = basis;
  h.value_bytes = value_bytes;
  h.flags = flags;
  h.rank = rank;
  h.world = world;
  h.n_blocks = n_blocks;
  h.n_values = n_values;
  h.keys_offset = sizeof(ShardHeader);
  h.values_offset = (h.keys_offset + n_blocks * sizeof(BlockRec) + 63) / 64 * 64;
  return h;
}

namespace {
struct FileCloser {
  void operator()(FILE* f) const {
    if (f) std::fclose(f);
  }
};
using File = std::unique_ptr<FILE, FileCloser>;
}  // namespace

BlockSet read_shard(const std::string& path, ShardHeader* out_hdr) {
  File f(std::fopen(path.c_str(), "rb"));
  if (!f) data("cannot open file: " + path);
  ShardHeader h;
  if (std::fread(&h, sizeof h, 1, f.get()) != 1 || std::memcmp(h.magic, "ESGBLKS1", 8) != 0)
    data("not a block shard: " + path);
  if (h.version != 1) data("unsupported block shard version: " + path);
  if (h.value_bytes != 4 && h.value_bytes != 8) data("bad value width in block shard: " + path);
  if (h.keys_offset != sizeof(ShardHeader) || h.values_offset < h.keys_offset + h.n_blocks * sizeof(BlockRec))
    data("bad section offsets in block shard: " + path);
  BlockSet s;
  s.keys.resize(h.n_blocks);
  if (h.n_blocks && std::fread(s.keys.data(), sizeof(BlockRec), h.n_blocks, f.get()) != h.n_blocks)
    data("truncated block shard: " + path);
  s.off.resize(h.n_blocks + 1);
  s.off[0] = 0;
  for (uint64_t b = 0; b < h.n_blocks; ++b) {
    if (s.keys[b].rows < 1 || s.keys[b].cols < 1) data("bad block shape in shard: " + path);
    s.off[b + 1] = s.off[b] + (int64_t)s.keys[b].rows * s.keys[b].cols;
  }
  if ((uint64_t)s.off[h.n_blocks] != h.n_values) data("block shapes do not add up to the value count: " + path);
  if (std::fseek(f.get(), (long)h.values_offset, SEEK_SET) != 0) data("truncated block shard: " + path);
  s.values.resize(h.n_values);
  if (h.value_bytes == 8) {
    if (h.n_values && std::fread(s.values.data(), 8, h.n_values, f.get()) != h.n_values)
      data("truncated block shard: " + path);
  } else {
    std::vector<float> v(h.n_values);
    if (h.n_values && std::fread(v.data(), 4, h.n_values, f.get()) != h.n_values)
      data("truncated block shard: " + path);
    for (uint64_t k = 0; k < h.n_values; ++k) s.values[k] = v[k];
  }
  if (out_hdr) *out_hdr = h;
  return s;
}

void write_blocks_text(const std::string& path, const std::vector<const BlockSet*>& sets) {
  struct Ref {
    const BlockRec* k;
    uint32_t set;
    int64_t idx;
  };
  std::vector<Ref> refs;
  size_t total = 0;
  for (const auto* s : sets) total += s->keys.size();
  refs.reserve(total);
  for (uint32_t si = 0; si < sets.size(); ++si)
    for (int64_t b = 0; b < (int64_t)sets[si]->keys.size(); ++b) refs.push_back({&sets[si]->keys[b], si, b});
  auto key = [](const BlockRec& r) { return std::array<int32_t, 5>{r.i, r.j, r.ix, r.iy, r.iz}; };
  // BlockKey order (i, j, image lexicographic); equal keys keep set order,
  // and the last one wins
  std::stable_sort(refs.begin(), refs.end(), [&](const Ref& a, const Ref& b) { return key(*a.k) < key(*b.k); });
  File f(std::fopen(path.c_str(), "wb"));
  if (!f) data("cannot open file for writing: " + path);
  std::vector<char> buf;
  buf.reserve(1 << 20);
  char tmp[64];
  auto flush = [&] {
    if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), f.get()) != buf.size()) data("write failed: " + path);
    buf.clear();
  };
  for (size_t r = 0; r < refs.size(); ++r) {
    if (r + 1 < refs.size() && key(*refs[r + 1].k) == key(*refs[r].k)) continue;
    const BlockRec& k = *refs[r].k;
    const BlockSet& s = *sets[refs[r].set];
    int n = std::snprintf(tmp, sizeof tmp, "%d %d %d %d %d %d %d", k.i, k.j, k.ix, k.iy, k.iz, (int)k.rows,
                          (int)k.cols);
    buf.insert(buf.end(), tmp, tmp + n);
    for (int64_t q = s.off[refs[r].idx]; q < s.off[refs[r].idx + 1]; ++q) {
      n = std::snprintf(tmp, sizeof tmp, " %.17g", s.values[q]);
      buf.insert(buf.end(), tmp, tmp + n);
    }
    buf.push_back('\n');
    if (buf.size() > (1 << 20)) flush();
  }
  flush();
}

// block_matrix.cpp:109-128 read_blocks: one block per line
// "i j ix iy iz rows cols v...", blank lines and '#' comments skipped, values
// parsed as std::istream does; malformed lines, bad shapes, short value lists
// and duplicate keys are data errors with the line number.  Blocks come back
// in BlockKey order (the std::map of the reference).
BlockSet read_blocks_text(const std::string& path) {
  std::ifstream in(path);
  if (!in) data("cannot open file: " + path);
  std::map<std::array<int32_t, 5>, std::pair<std::array<int32_t, 2>, std::vector<double>>> bm;
  std::string line;
  long lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ss(line);
    int32_t k[5];
    long rows = 0, cols = 0;
    if (!(ss >> k[0] >> k[1] >> k[2] >> k[3] >> k[4] >> rows >> cols))
      data("expected 'i j ix iy iz rows cols values...' (line " + std::to_string(lineno) + ")");
    if (rows < 1 || cols < 1 || rows > 65535 || cols > 65535)
      data("bad block shape (line " + std::to_string(lineno) + ")");
    std::vector<double> v((size_t)rows * cols);
    for (double& x : v)
      if (!(ss >> x)) data("short block value list (line " + std::to_string(lineno) + ")");
    const std::array<int32_t, 5> key{k[0], k[1], k[2], k[3], k[4]};
    if (!bm.emplace(key, std::make_pair(std::array<int32_t, 2>{(int32_t)rows, (int32_t)cols}, std::move(v))).second)
      data("duplicate block key (line " + std::to_string(lineno) + ")");
  }
  BlockSet s;
  s.off.push_back(0);
  for (auto& [key, blk] : bm) {
    s.keys.push_back({key[0], key[1], key[2], key[3], key[4], (uint16_t)blk.first[0], (uint16_t)blk.first[1]});
    s.values.insert(s.values.end(), blk.second.begin(), blk.second.end());
    s.off.push_back((int64_t)s.values.size());
  }
  return s;
}

}  // namespace esg
