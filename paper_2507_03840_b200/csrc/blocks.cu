// blocks.cu -- block-sparse export of the last forward (SURVEY §8 row a17 and
// §8(f) 1).
//
// Reference path: Network::assemble_blocks (network.h:168-184) builds a
// std::map of heap matrices via fill_block (network.h:296-315), the ranks'
// maps are serialised to text and gathered on rank 0 (model_run.cpp:103-120),
// and blocks_to_uncoupled (block_matrix.cpp:66-88, to_block
// clebsch_gordan.cpp:157-170) converts every shell-pair rectangle.  Here the
// blocks are produced on the device straight from the head outputs into a
// flat layout (keys + concatenated row-major values, blocks_io.h), streamed
// to per-rank shard files through two pinned buffers so the D2H copy and the
// file write of chunk c overlap the kernels of chunk c+1.
//
// Values are bit-exact against the CPU restatement: coupled values are the
// fp32 heads widened; uncoupled values sum the coupling terms per L segment
// then across L in to_block's order with no FMA contraction (__dmul_rn /
// __dadd_rn), and the coupling tables are built by the same construction as
// the oracle's (host.cpp coupling_matrix).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <array>
#include <algorithm>
#include <memory>

#include "blocks_io.h"
#include "device_model.h"

namespace esg {

// Per basis mode: for every species-slot pair p = slot_a * S + slot_b the
// block shape and, per block element (row-major), its terms (head index,
// coefficient) in to_block order; bit 31 of a term index marks the first
// term of an L segment.
// Exactly-zero coefficients are dropped: the running sums start at +0 and
// never become -0 under round-to-nearest, so adding a zero product cannot
// change them -- the result is bit-identical for finite heads (a NaN/Inf head
// no longer reaches elements whose coefficient on it is zero).
struct __align__(16) BlockTerm {
  double c;
  uint32_t idx;  // head index | kSegStart on the first kept term of an L segment
  uint32_t pad;
};

struct BlockTables {
  int S = 0, max_elem = 1;
  int *nelem = nullptr, *rows = nullptr, *cols = nullptr, *ptr0 = nullptr, *eptr = nullptr;
  BlockTerm* terms = nullptr;
};

struct BlockState {
  BlockTables* bt[2] = {nullptr, nullptr};  // coupled, uncoupled
  int64_t* off = nullptr;                   // per item value offset, n_items + 1
  size_t cap_off = 0;
  int64_t n_items = 0, n_values = 0;
  int max_elem = 1;
  // chunk pipeline: two device and two pinned host staging buffers
  void* dbuf[2] = {nullptr, nullptr};
  void* hbuf[2] = {nullptr, nullptr};
  size_t cap_buf = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
};

namespace {

constexpr uint32_t kSegStart = 0x80000000u;
constexpr int kTileItems = 64;        // items per CTA in the value kernel
constexpr size_t kChunkBytes = 64 << 20;  // staging buffer size

template <typename T>
T* upload(const std::vector<T>& h, cudaStream_t st) {
  T* p = nullptr;
  if (h.empty()) return p;
  ESG_CUDA(cudaMalloc(&p, h.size() * sizeof(T)));
  ESG_CUDA(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return p;
}

__device__ __forceinline__ int item_pair(int64_t it, int n_owned, const int* __restrict__ row_slot,
                                         const int* __restrict__ src_row, const int* __restrict__ dst_row, int S) {
  if (it < n_owned) {
    const int s = row_slot[it];
    return s * S + s;
  }
  const int64_t k = it - n_owned;
  return row_slot[src_row[k]] * S + row_slot[dst_row[k]];
}

__global__ void k_item_nelem(int64_t n_items, int n_owned, const int* __restrict__ row_slot,
                             const int* __restrict__ src_row, const int* __restrict__ dst_row, int S,
                             const int* __restrict__ nelem, int64_t* __restrict__ out) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it > n_items) return;
  out[it] = it < n_items ? nelem[item_pair(it, n_owned, row_slot, src_row, dst_row, S)] : 0;
}

// out[c] = off[min(c * per, n)] for c = 0..nc
__global__ void k_chunk_bounds(const int64_t* __restrict__ off, int64_t per, int64_t n, int nc,
                               int64_t* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nc) return;
  const int64_t i = (int64_t)c * per;
  out[c] = off[i < n ? i : n];
}

// keys of items [a, a + n): (g, g, 0) for owned atoms, (src, dst, shift)
// for edges (network.h:172-182); shapes from the species pair
__global__ void k_block_keys(int64_t a, int64_t n, int n_owned, const int* __restrict__ row_global,
                             const int* __restrict__ row_slot, const int* __restrict__ src_row,
                             const int* __restrict__ dst_row, const uint32_t* __restrict__ eshift, int S,
                             const int* __restrict__ rows, const int* __restrict__ cols, BlockRec* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t it = a + t;
  BlockRec r;
  if (it < n_owned) {
    r.i = r.j = row_global[it];
    r.ix = r.iy = r.iz = 0;
  } else {
    const int64_t k = it - n_owned;
    r.i = row_global[src_row[k]];
    r.j = row_global[dst_row[k]];
    const uint32_t s = eshift[k];
    r.ix = int((s >> 20) & 1023u) - 512;
    r.iy = int((s >> 10) & 1023u) - 512;
    r.iz = int(s & 1023u) - 512;
  }
  const int p = item_pair(it, n_owned, row_slot, src_row, dst_row, S);
  r.rows = (uint16_t)rows[p];
  r.cols = (uint16_t)cols[p];
  out[t] = r;
}

__device__ __forceinline__ double uncoupled_value(const float* __restrict__ row, int e, const int* __restrict__ eptr,
                                                  const BlockTerm* __restrict__ terms) {
  // to_block: flat = sum over L of C_L^T c_L, each product summed over r
  // from zero, then added to the running total in L order
  double tot = 0.0, acc = 0.0;
  const int q0 = eptr[e], q1 = eptr[e + 1];
  for (int q = q0; q < q1; ++q) {
    const BlockTerm t = terms[q];
    if ((t.idx & kSegStart) && q > q0) {
      tot = __dadd_rn(tot, acc);
      acc = 0.0;
    }
    acc = __dadd_rn(acc, __dmul_rn(t.c, (double)row[t.idx & ~kSegStart]));
  }
  return __dadd_rn(tot, acc);
}

// Values of items [a, a + n) written contiguously from out[0] (= the value
// offset of item a).  One CTA per tile of kTileItems items: the tile's
// value -> item map is built in shared memory (one byte per value), then the
// threads walk the tile's values in order (coalesced stores).
template <bool COUPLED, typename VT>
__global__ void __launch_bounds__(256) k_block_values(int64_t a, int64_t n, int n_owned, const float* __restrict__ node_out,
                                                      const float* __restrict__ edge_out, int out_len,
                                                      const int* __restrict__ row_slot, const int* __restrict__ src_row,
                                                      const int* __restrict__ dst_row, int S,
                                                      const int64_t* __restrict__ off, const int* __restrict__ cols,
                                                      const int* __restrict__ ptr0, const int* __restrict__ eptr,
                                                      const BlockTerm* __restrict__ terms, int symmetrize,
                                                      VT* __restrict__ out) {
  extern __shared__ uint8_t s_item[];  // kTileItems * max_elem bytes
  __shared__ int64_t s_off[kTileItems + 1];
  __shared__ int s_base[kTileItems];  // ptr0 of the item's species pair
  __shared__ int s_cols[kTileItems];
  __shared__ const float* s_row[kTileItems];
  const int64_t t0 = a + (int64_t)blockIdx.x * kTileItems;
  const int64_t left = a + n - t0;
  const int nt = left < kTileItems ? (int)left : kTileItems;
  if (nt <= 0) return;
  for (int i = threadIdx.x; i <= nt; i += blockDim.x) {
    s_off[i] = off[t0 + i];
    if (i < nt) {
      const int64_t it = t0 + i;
      const int p = item_pair(it, n_owned, row_slot, src_row, dst_row, S);
      s_base[i] = ptr0[p];
      s_cols[i] = cols[p];
      s_row[i] = it < n_owned ? node_out + it * out_len : edge_out + (it - n_owned) * out_len;
    }
  }
  __syncthreads();
  const int64_t v0 = s_off[0];
  const int nv = (int)(s_off[nt] - v0);
  for (int i = threadIdx.x >> 5; i < nt; i += blockDim.x >> 5)
    for (int j = (int)(s_off[i] - v0) + (threadIdx.x & 31); j < (int)(s_off[i + 1] - v0); j += 32) s_item[j] = (uint8_t)i;
  __syncthreads();
  VT* o = out + (v0 - off[a]);
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    const int i = s_item[v];
    const int j = v - (int)(s_off[i] - v0);
    const float* row = s_row[i];
    const int e = s_base[i] + j;
    double val;
    if (COUPLED) {
      val = (double)row[terms[e].idx & ~kSegStart];  // one term per element: eptr[e] == e
    } else {
      val = uncoupled_value(row, e, eptr, terms);
      if (symmetrize && t0 + i < n_owned) {  // block_matrix.cpp:84-85: 0.5 (ub + ub^T) on (i, i, 0)
        const int nc = s_cols[i], r = j / nc, c = j % nc;
        if (r != c) val = __dmul_rn(0.5, __dadd_rn(val, uncoupled_value(row, s_base[i] + c * nc + r, eptr, terms)));
      }
    }
    o[v] = (VT)val;
  }
}

BlockTables* build_tables(const esg_model* M, bool coupled, cudaStream_t st) {
  const auto& sl = M->species_list;
  const int S = (int)sl.size();
  std::vector<int> nelem(S * S), rows(S * S), cols(S * S), ptr0(S * S), eptr{0};
  std::vector<BlockTerm> tl_all;
  std::map<std::array<int, 3>, std::vector<double>> cg;
  int max_elem = 1;
  for (int sa = 0; sa < S; ++sa)
    for (int sb = 0; sb < S; ++sb) {
      const int za = sl[sa], zb = sl[sb], p = sa * S + sb;
      const auto& sha = M->basis.shells.at(za);
      const auto& shb = M->basis.shells.at(zb);
      const int na = M->basis.n_orb(za), nb = M->basis.n_orb(zb);
      std::vector<std::vector<std::pair<uint32_t, double>>> terms((size_t)na * nb);
      for (size_t a = 0; a < sha.size(); ++a)
        for (size_t b = 0; b < shb.size(); ++b) {
          const int la = sha[a], lb = shb[b], db = 2 * lb + 1, da = 2 * la + 1;
          const int oa = M->basis.off(za, (int)a), ob = M->basis.off(zb, (int)b);
          auto el = [&](int q) -> auto& { return terms[(size_t)(oa + q / db) * nb + ob + q % db]; };
          int pos = 0;  // fill_block: coupled segments row-major in the rectangle
          for (int L = std::abs(la - lb); L <= la + lb; ++L) {
            const int seg = M->heads.segment((int)a, (int)b, L);
            if (coupled) {
              for (int r = 0; r < 2 * L + 1; ++r, ++pos) el(pos).push_back({(uint32_t)(seg + r) | kSegStart, 1.0});
              continue;
            }
            auto key = std::array<int, 3>{la, lb, L};
            if (!cg.count(key)) cg[key] = coupling_matrix(la, lb, L);
            const auto& C = cg[key];
            for (int q = 0; q < da * db; ++q) {
              bool first = true;
              for (int r = 0; r < 2 * L + 1; ++r) {
                const double c = C[(size_t)r * da * db + q];
                if (c == 0.0) continue;
                el(q).push_back({(uint32_t)(seg + r) | (first ? kSegStart : 0u), c});
                first = false;
              }
            }
          }
        }
      nelem[p] = na * nb;
      rows[p] = na;
      cols[p] = nb;
      ptr0[p] = (int)eptr.size() - 1;
      max_elem = std::max(max_elem, na * nb);
      for (const auto& tl : terms) {
        for (const auto& t : tl) tl_all.push_back({t.second, t.first, 0u});
        eptr.push_back((int)tl_all.size());
      }
    }
  auto* T = new BlockTables;
  T->S = S;
  T->max_elem = max_elem;
  T->nelem = upload(nelem, st);
  T->rows = upload(rows, st);
  T->cols = upload(cols, st);
  T->ptr0 = upload(ptr0, st);
  T->eptr = upload(eptr, st);
  T->terms = upload(tl_all, st);
  ESG_CUDA(cudaStreamSynchronize(st));
  return T;
}

void free_tables(BlockTables* T) {
  if (!T) return;
  for (void* p : {(void*)T->nelem, (void*)T->rows, (void*)T->cols, (void*)T->ptr0, (void*)T->eptr, (void*)T->terms})
    free_ptr(p);
  delete T;
}

BlockState& state(esg_model* M) {
  DeviceModel* D = M->dev;
  if (!D || !D->prepared) usage("blocks requested before prepare");
  if (!D->blk) {
    D->blk = new BlockState;
    ESG_CUDA(cudaEventCreate(&D->blk->ev[0]));
    ESG_CUDA(cudaEventCreate(&D->blk->ev[1]));
    ESG_CUDA(cudaEventCreate(&D->blk->t0));
    ESG_CUDA(cudaEventCreate(&D->blk->t1));
  }
  BlockState& B = *D->blk;
  cudaStream_t st = M->ctx->stream;
  for (int c = 0; c < 2; ++c)
    if (!B.bt[c]) B.bt[c] = build_tables(M, c == 0, st);
  if (!D->blk_ready) {
    // per-item value counts, exclusive scan -> offsets (n_items + 1)
    B.n_items = D->n_owned + D->n_edges;
    if (B.cap_off < (size_t)B.n_items + 1) {
      free_ptr(B.off);
      B.cap_off = B.n_items + 1;
      ESG_CUDA(cudaMalloc(&B.off, B.cap_off * sizeof(int64_t)));
    }
    int64_t* cnt = nullptr;
    ESG_CUDA(cudaMalloc(&cnt, (B.n_items + 1) * sizeof(int64_t)));
    const BlockTables& T = *B.bt[1];
    k_item_nelem<<<(unsigned)((B.n_items + 256) / 256), 256, 0, st>>>(B.n_items, D->n_owned, D->row_slot, D->src_row,
                                                                       D->dst_row, T.S, T.nelem, cnt);
    ++M->ctx->launches;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, B.off, B.n_items + 1, st);
    void* tmp = nullptr;
    ESG_CUDA(cudaMalloc(&tmp, tb));
    ESG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, B.off, B.n_items + 1, st));
    ESG_CUDA(cudaMemcpyAsync(&B.n_values, B.off + B.n_items, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    ESG_CUDA(cudaStreamSynchronize(st));
    free_ptr(tmp);
    free_ptr(cnt);
    B.max_elem = T.max_elem;
    D->blk_ready = true;
  }
  return B;
}

void launch_keys(esg_model* M, BlockState& B, int64_t a, int64_t n, BlockRec* out) {
  DeviceModel* D = M->dev;
  if (n <= 0) return;
  const BlockTables& T = *B.bt[1];
  k_block_keys<<<(unsigned)((n + 255) / 256), 256, 0, M->ctx->stream>>>(a, n, D->n_owned, D->row_global, D->row_slot,
                                                                         D->src_row, D->dst_row, D->eshift, T.S, T.rows,
                                                                         T.cols, out);
  ++M->ctx->launches;
}

void launch_values(esg_model* M, BlockState& B, int basis, bool sym, int vb, int64_t a, int64_t n, void* out) {
  DeviceModel* D = M->dev;
  if (n <= 0) return;
  const BlockTables& T = *B.bt[basis];
  const unsigned grid = (unsigned)((n + kTileItems - 1) / kTileItems);
  const size_t smem = (size_t)kTileItems * T.max_elem;
  if (smem > 48 * 1024) usage("block too large for the export kernel (max 768 elements per block)");
  cudaStream_t st = M->ctx->stream;
  const int ol = M->heads.out_len;
#define ESG_BV(C, VT)                                                                                              \
  k_block_values<C, VT><<<grid, 256, smem, st>>>(a, n, D->n_owned, D->node_out, D->edge_out, ol, D->row_slot,         \
                                              D->src_row, D->dst_row, T.S, B.off, T.cols, T.ptr0, T.eptr, T.terms, \
                                              sym ? 1 : 0, (VT*)out)
  if (basis == 0) {
    if (vb == 8) ESG_BV(true, double);
    else ESG_BV(true, float);
  } else {
    if (vb == 8) ESG_BV(false, double);
    else ESG_BV(false, float);
  }
#undef ESG_BV
  ++M->ctx->launches;
  ESG_CUDA(cudaGetLastError());
}

void check_args(int basis, bool sym, int vb) {
  if (basis != 0 && basis != 1) usage("basis must be ESG_BLOCKS_COUPLED or ESG_BLOCKS_UNCOUPLED");
  if (sym && basis != 1) usage("on-site symmetrisation applies to uncoupled blocks only");
  if (vb != 4 && vb != 8) usage("value width must be 4 or 8 bytes");
}

// Items in chunks whose keys and values fit one staging buffer; each chunk
// is computed on the device, copied to pinned memory and handed to sink
// while the next chunk computes.  keys: true for the key table, false for
// the values.
// ESG_BLOCK_CHUNK_BYTES overrides the staging size (tests use small chunks
// to exercise the pipeline)
size_t chunk_bytes() {
  const char* e = std::getenv("ESG_BLOCK_CHUNK_BYTES");
  const long long v = e ? std::atoll(e) : 0;
  return v >= 4096 ? (size_t)v : kChunkBytes;
}

template <class Sink>
void stream_items(esg_model* M, BlockState& B, bool keys, int basis, bool sym, int vb, Sink sink) {
  cudaStream_t st = M->ctx->stream;
  const size_t cb = chunk_bytes();
  if (B.cap_buf != cb) {
    for (int c = 0; c < 2; ++c) {
      free_ptr(B.dbuf[c]);
      if (B.hbuf[c]) cudaFreeHost(B.hbuf[c]);
      ESG_CUDA(cudaMalloc(&B.dbuf[c], cb));
      ESG_CUDA(cudaMallocHost(&B.hbuf[c], cb));
    }
    B.cap_buf = cb;
  }
  const int64_t per = std::max<int64_t>(1, (int64_t)(cb / std::max<size_t>(sizeof(BlockRec), (size_t)vb * B.max_elem)));
  const int nc = (int)((B.n_items + per - 1) / per);
  if (nc == 0) return;
  std::vector<int64_t> vb_at(nc + 1);  // value offset at each chunk boundary
  if (!keys) {
    int64_t* d = nullptr;
    ESG_CUDA(cudaMalloc(&d, (nc + 1) * sizeof(int64_t)));
    k_chunk_bounds<<<(nc + 256) / 256, 256, 0, st>>>(B.off, per, B.n_items, nc, d);
    ++M->ctx->launches;
    ESG_CUDA(cudaMemcpyAsync(vb_at.data(), d, (nc + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    ESG_CUDA(cudaStreamSynchronize(st));
    free_ptr(d);
  }
  auto bytes = [&](int c) -> size_t {
    const int64_t a = (int64_t)c * per, b = std::min(B.n_items, a + per);
    return keys ? (size_t)(b - a) * sizeof(BlockRec) : (size_t)(vb_at[c + 1] - vb_at[c]) * vb;
  };
  for (int c = 0; c <= nc; ++c) {
    if (c < nc) {
      const int64_t a = (int64_t)c * per, n = std::min(B.n_items, a + per) - a;
      if (keys) launch_keys(M, B, a, n, (BlockRec*)B.dbuf[c & 1]);
      else launch_values(M, B, basis, sym, vb, a, n, B.dbuf[c & 1]);
      ESG_CUDA(cudaMemcpyAsync(B.hbuf[c & 1], B.dbuf[c & 1], bytes(c), cudaMemcpyDeviceToHost, st));
      ESG_CUDA(cudaEventRecord(B.ev[c & 1], st));
    }
    if (c > 0) {
      ESG_CUDA(cudaEventSynchronize(B.ev[(c - 1) & 1]));
      sink(B.hbuf[(c - 1) & 1], bytes(c - 1));
    }
  }
}

}  // namespace

void blocks_free(DeviceModel* D) {
  BlockState* B = D->blk;
  if (!B) return;
  free_tables(B->bt[0]);
  free_tables(B->bt[1]);
  free_ptr(B->off);
  for (int c = 0; c < 2; ++c) {
    free_ptr(B->dbuf[c]);
    if (B->hbuf[c]) cudaFreeHost(B->hbuf[c]);
    if (B->ev[c]) cudaEventDestroy(B->ev[c]);
  }
  if (B->t0) cudaEventDestroy(B->t0);
  if (B->t1) cudaEventDestroy(B->t1);
  delete B;
  D->blk = nullptr;
  D->blk_ready = false;
}

void blocks_count(esg_model* M, int64_t* n_blocks, int64_t* n_values) {
  BlockState& B = state(M);
  if (n_blocks) *n_blocks = B.n_items;
  if (n_values) *n_values = B.n_values;
}

void blocks_export(esg_model* M, int basis, bool sym, BlockRec* keys, double* values) {
  check_args(basis, sym, 8);
  BlockState& B = state(M);
  if (keys) {
    char* at = (char*)keys;
    stream_items(M, B, true, basis, sym, 8, [&](const void* h, size_t n) {
      std::memcpy(at, h, n);
      at += n;
    });
  }
  if (values) {
    char* at = (char*)values;
    stream_items(M, B, false, basis, sym, 8, [&](const void* h, size_t n) {
      std::memcpy(at, h, n);
      at += n;
    });
  }
}

void blocks_export_device(esg_model* M, int basis, bool sym, int vb, void* d_keys, void* d_values, float* kernel_ms) {
  check_args(basis, sym, vb);
  BlockState& B = state(M);
  cudaStream_t st = M->ctx->stream;
  ESG_CUDA(cudaEventRecord(B.t0, st));
  if (d_keys) launch_keys(M, B, 0, B.n_items, (BlockRec*)d_keys);
  if (d_values) launch_values(M, B, basis, sym, vb, 0, B.n_items, d_values);
  ESG_CUDA(cudaEventRecord(B.t1, st));
  ESG_CUDA(cudaStreamSynchronize(st));
  if (kernel_ms) ESG_CUDA(cudaEventElapsedTime(kernel_ms, B.t0, B.t1));
}

void blocks_write_shard(esg_model* M, const char* path, int basis, bool sym, int vb) {
  check_args(basis, sym, vb);
  BlockState& B = state(M);
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), &std::fclose);
  if (!f) data(std::string("cannot open file for writing: ") + path);
  const ShardHeader h = shard_header((uint32_t)basis, (uint32_t)vb, sym ? 1u : 0u, (uint32_t)M->ctx->rank,
                                     (uint32_t)M->ctx->world, (uint64_t)B.n_items, (uint64_t)B.n_values);
  auto put = [&](const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f.get()) != n) data(std::string("write failed: ") + path);
  };
  put(&h, sizeof h);
  stream_items(M, B, true, basis, sym, vb, put);
  const std::vector<char> pad(h.values_offset - h.keys_offset - h.n_blocks * sizeof(BlockRec), 0);
  put(pad.data(), pad.size());
  stream_items(M, B, false, basis, sym, vb, put);
  if (std::fflush(f.get()) != 0) data(std::string("write failed: ") + path);
}

// Network::build_targets (network.h:187-214) with encode_target
// (network.h:318-343, clebsch_gordan.cpp:142-155 to_coupled): for every item
// of the prepared view whose key has a target block, each shell-pair
// rectangle is mapped to its coupled coefficients c_L = C_L . flat (sums in
// ascending element order) and placed at the item's head slots; mask 1 there.
int64_t build_targets(esg_model* M, int64_t n_blocks, const BlockRec* keys, const double* values, float* node_t,
                      uint8_t* node_m, float* edge_t, uint8_t* edge_m) {
  BlockState& B = state(M);
  DeviceModel* D = M->dev;
  const int ol = M->heads.out_len;
  std::vector<BlockRec> items(B.n_items);
  blocks_export(M, ESG_BLOCKS_UNCOUPLED, false, items.data(), nullptr);
  std::vector<int32_t> src(D->n_edges), dst(D->n_edges);  // the view's endpoint rows (species)
  if (D->n_edges) {
    d2h_small(M->ctx, src.data(), D->src_row, sizeof(int32_t) * D->n_edges);
    d2h_small(M->ctx, dst.data(), D->dst_row, sizeof(int32_t) * D->n_edges);
  }
  struct KeyHash {
    size_t operator()(const std::array<int32_t, 5>& k) const {
      size_t h = 1469598103934665603ull;
      for (int32_t v : k) h = (h ^ (uint32_t)v) * 1099511628211ull;
      return h;
    }
  };
  std::unordered_map<std::array<int32_t, 5>, int64_t, KeyHash> where;
  where.reserve((size_t)n_blocks * 2);
  std::vector<int64_t> off((size_t)n_blocks + 1, 0);
  for (int64_t b = 0; b < n_blocks; ++b) {
    const BlockRec& k = keys[b];
    if (k.rows < 1 || k.cols < 1) data("bad target block shape");
    off[b + 1] = off[b] + (int64_t)k.rows * k.cols;
    where[{k.i, k.j, k.ix, k.iy, k.iz}] = b;  // BlockMatrix keeps one block per key
  }
  std::map<std::array<int, 3>, std::vector<double>> cg;
  auto coupling_of = [&](int la, int lb, int L) -> const std::vector<double>& {
    auto key = std::array<int, 3>{la, lb, L};
    auto it = cg.find(key);
    if (it == cg.end()) it = cg.emplace(key, coupling_matrix(la, lb, L)).first;
    return it->second;
  };
  int64_t count = 0;
  for (int64_t it = 0; it < B.n_items; ++it) {
    const BlockRec& k = items[it];
    const auto f = where.find({k.i, k.j, k.ix, k.iy, k.iz});
    const bool node = it < D->n_owned;
    float* row = node ? (node_t ? node_t + it * ol : nullptr) : (edge_t ? edge_t + (it - D->n_owned) * ol : nullptr);
    uint8_t* mask = node ? (node_m ? node_m + it * ol : nullptr) : (edge_m ? edge_m + (it - D->n_owned) * ol : nullptr);
    if (row) std::fill(row, row + ol, 0.f);
    if (mask) std::fill(mask, mask + ol, (uint8_t)0);
    if (f == where.end()) continue;
    const int64_t b = f->second;
    if (keys[b].rows != k.rows || keys[b].cols != k.cols) data("target block shape does not match the species basis");
    const double* blk = values + off[b];
    const int nb = k.cols;
    const int64_t e = it - D->n_owned;
    const int zi = node ? D->row_species[it] : D->row_species[src[e]];
    const int zj = node ? D->row_species[it] : D->row_species[dst[e]];
    const auto& sha = M->basis.shells.at(zi);
    const auto& shb = M->basis.shells.at(zj);
    for (size_t a = 0; a < sha.size(); ++a)
      for (size_t c = 0; c < shb.size(); ++c) {
        const int la = sha[a], lb = shb[c], da = 2 * la + 1, db = 2 * lb + 1;
        const int oa = M->basis.off(zi, (int)a), ob = M->basis.off(zj, (int)c);
        std::vector<double> flat((size_t)da * db);
        for (int i = 0; i < da; ++i)
          for (int j = 0; j < db; ++j) flat[(size_t)i * db + j] = blk[(size_t)(oa + i) * nb + ob + j];
        for (int L = std::abs(la - lb); L <= la + lb; ++L) {
          const auto& C = coupling_of(la, lb, L);
          const int seg = M->heads.segment((int)a, (int)c, L);
          for (int r = 0; r < 2 * L + 1; ++r) {
            double acc = 0.0;
            for (int q = 0; q < da * db; ++q) acc += C[(size_t)r * da * db + q] * flat[q];
            if (row) row[seg + r] = static_cast<float>(acc);
            if (mask) mask[seg + r] = 1;
            ++count;
          }
        }
      }
  }
  return count;
}

void blocks_write_text(esg_model* M, const char* path, int basis, bool sym) {
  check_args(basis, sym, 8);
  BlockState& B = state(M);
  BlockSet s;
  s.keys.resize(B.n_items);
  s.values.resize(B.n_values);
  blocks_export(M, basis, sym, s.keys.data(), s.values.data());
  s.off.resize(B.n_items + 1);
  s.off[0] = 0;
  for (int64_t b = 0; b < B.n_items; ++b) s.off[b + 1] = s.off[b] + (int64_t)s.keys[b].rows * s.keys[b].cols;
  write_blocks_text(path, {&s});
}

}  // namespace esg
