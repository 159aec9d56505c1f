// blocks_io.h -- the flat block-sparse shard format and the reference's text
// form.  Host-only; no CUDA types.
//
// Shard file (little-endian), one per rank, replacing the std::map
// BlockMatrix and the text gather to rank 0 (model_run.cpp:103-120):
//   0   char[8]  "ESGBLKS1"
//   8   u32      version (1)
//   12  u32      basis (0 coupled, 1 uncoupled)
//   16  u32      value bytes (8 fp64, 4 fp32)
//   20  u32      flags (bit 0: on-site blocks symmetrised)
//   24  u32      rank, 28 u32 world
//   32  u64      n_blocks, 40 u64 n_values
//   48  u64      keys offset (64), 56 u64 values offset (64-byte aligned)
//   keys:   n_blocks x BlockRec (24 B: i, j, ix, iy, iz as i32; rows, cols as u16)
//   values: n_values values, each block row-major, blocks in key-table order
// Key-table order is the rank view's item order: owned atoms ascending
// (key (g, g, 0)), then owned edges in global edge order (key (src, dst,
// shift)).  The text writer orders by BlockKey (block_matrix.h:21-25).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace esg {

struct BlockRec {
  int32_t i, j, ix, iy, iz;
  uint16_t rows, cols;
};
static_assert(sizeof(BlockRec) == 24, "BlockRec is a 24-byte record");

struct ShardHeader {
  char magic[8];
  uint32_t version, basis, value_bytes, flags, rank, world;
  uint64_t n_blocks, n_values, keys_offset, values_offset;
};
static_assert(sizeof(ShardHeader) == 64, "shard header is 64 bytes");

ShardHeader shard_header(uint32_t basis, uint32_t value_bytes, uint32_t flags, uint32_t rank, uint32_t world,
                         uint64_t n_blocks, uint64_t n_values);

// One block source for the text writer: keys, per-block value offsets and
// fp64 values (shards with fp32 values are widened on read).
struct BlockSet {
  std::vector<BlockRec> keys;
  std::vector<int64_t> off;  // n_blocks + 1
  std::vector<double> values;
};

BlockSet read_shard(const std::string& path, ShardHeader* hdr = nullptr);

// block_matrix.cpp:90-101 write_blocks over the union of sets: one line per
// block "i j ix iy iz rows cols v..." with 17 significant digits, blocks in
// BlockKey order; a key present in several sets keeps the last set's block
// (gather_blocks' insert_or_assign, model_run.cpp:108-118).
void write_blocks_text(const std::string& path, const std::vector<const BlockSet*>& sets);

// block_matrix.cpp:109-128 read_blocks_file
BlockSet read_blocks_text(const std::string& path);

}  // namespace esg
