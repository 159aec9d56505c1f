// device_model.h -- the device state of one model (weights, the prepared
// view, feature tables, chunk scratch, halo buffers and training buffers).
// Shared by model.cu (forward) and train.cu (backward).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

#include "esg_internal.h"
#include "model_kernels.cuh"

namespace esg {

struct TrainState;  // train.cu

// one (order block, <= 256-output tile) of a tf32x3 tensor-core linear
// (tf32_gemm.cu): A columns [a_col, a_col + K), C columns [c_col, c_col + N),
// B image chunks at byte b_off
struct TcTile {
  int a_col, c_col, K, N;  // N: the MMA width (a multiple of 16)
  int n_valid;             // output columns actually stored (<= N)
  int64_t b_off;
};
// one output tile of a weight-gradient product (dw_tc.cu): g channels
// [goff, goff + nN) x x channels [xoff, xoff + nK) of an order block whose
// expanded gradient (N x K, row-major) starts at acc_off
struct DwTile {
  int goff, xoff, n0, k0, nN, nK, nKp, K;  // nKp: the MMA width (multiple of 16)
  int64_t acc_off;
};
int dw_tiles(int L, int E, int which, std::vector<DwTile>* tiles);
int64_t dw_part_floats(int n_tiles, int n_split);
void dw_tf32x3_launch(const float* g, int64_t ldg, const float* x, int64_t ldx, int64_t n_e, const DwTile* tiles,
                      int n_tiles, int split_e, float* part, double* acc, cudaStream_t st,
                      const float* gscale = nullptr, int gate_c2 = 0);
int64_t tf32_tiles(int L, int E, int kind, std::vector<TcTile>* tiles);
void tf32_pack(const float* params, int L, int E, int li, bool dx, const int64_t* off_a, const int64_t* off_b,
               uint8_t* img, cudaStream_t st);
// gate_c2 = 2E: lin2 with the gate of its operand fused into the A load
// (A holds ungated lin1 outputs); 0: plain product
void tf32_gemm_launch(const float* A, int64_t lda, int64_t n_rows, const uint8_t* img, const TcTile* tiles,
                      int n_tiles, float* C, int64_t ldc, cudaStream_t st, int gate_c2 = 0);

// Power-of-two scales of the fp16x3 chain (so2_f16x3.cu), per order m: the
// weight scales of lin1 / lin2 and ||W1_m||_inf (max row sum of |w|), which
// bounds lin1's output from the message bound
struct F16x3Scales {
  float w1[8], w2[8], w1inf[8];
};
bool so2_f16x3_available(int L, int E);
int64_t so2_f16x3_a1_tile_bytes(int L, int E);
int64_t so2_f16x3_w1_bytes(int L, int E);
int64_t so2_f16x3_w2_bytes(int L, int E);
int so2_f16x3_kofs(int m);
int so2_f16x3_ktot();
void so2_f16x3_launch(int L, int E, const uint8_t* A1, int64_t n_e, const uint8_t* W1, const uint8_t* W2,
                      const F16x3Scales& sc, const float* tmax, int edge_slot, float* Y, int gate, const float* att,
                      float* logits, cudaStream_t st);

struct DeviceModel {
  int L = 0, E = 0, H = 0;
  // weights (device)
  float* params = nullptr;  // raw flat parameters
  std::vector<float*> w1t, w2t;      // per block (2*layers): SIMT packed
  std::vector<uint16_t*> w1b, w2b;   // per block: tcgen05 bf16 packed
  std::vector<uint8_t*> w1f, w2f;    // per block: fp16x3 split images (so2_f16x3.cu)
  std::vector<F16x3Scales> f16sc;    // per block: their scales
  bool f16_stale = true;             // the images predate the current parameters
  bool f16x3 = true;                 // ESG_F16X3=0: fp32 linears on the tf32 GEMMs instead
  // |x| maxima of the feature tables for the fp16x3 scale bounds: [0] the
  // node table entering the current block, [1 + l] the edge table entering
  // layer l (written by the init / rotate_out kernels)
  float* tmax = nullptr;
  std::vector<float*> w1n, w2n;      // per block: expanded, not transposed (training dx = W^T g)
  bool weights_allocated = false;
  struct LinTile* lt[4] = {nullptr, nullptr, nullptr, nullptr};  // k_gemm_m tile lists (lin_kernels.cuh)
  int n_lt[4] = {0, 0, 0, 0};
  // fp32-accurate linears on the tensor cores (3xTF32): per kind (0 lin1,
  // 1 lin2, 2 lin2 dx, 3 lin1 dx) one B image per block and a shared tile list
  std::vector<uint8_t*> wtc[4];
  TcTile* tct[4] = {nullptr, nullptr, nullptr, nullptr};
  int n_tct[4] = {0, 0, 0, 0};
  bool tf32 = true;  // ESG_TF32=0 selects the CUDA-core SGEMM instead
  float* Hbuf = nullptr;  // fp32 path: lin1 output / gated operand of a chunk
  size_t cap_hbuf = 0;
  std::vector<int64_t> att_off;      // per layer offset into params
  float* embed = nullptr;            // per species slot x E
  float* head_w[2] = {nullptr, nullptr};  // node / edge: n_keys x E
  int* head_key = nullptr;   // per listed output: key index
  int* head_row = nullptr;   // per listed output: output index
  int* head_hptr = nullptr;  // per harmonic row: start of its outputs
  int64_t lift_off = 0;
  // prepared view
  bool prepared = false;
  int n_rows = 0, n_owned = 0;
  int64_t n_edges = 0;
  int* row_slot = nullptr;
  std::vector<int> row_species;
  int* src_row = nullptr;
  int* dst_row = nullptr;
  float* dir = nullptr;
  double* dist = nullptr;
  int64_t* seg = nullptr;  // n_owned + 1
  std::vector<int64_t> h_seg;
  std::vector<std::pair<int, int>> chunks;  // owned-row ranges, dst aligned
  // halo
  std::vector<esg::Neighbor> nbrs;
  int* send_rows = nullptr;
  int64_t n_send = 0;
  float* send_buf = nullptr;
  // tables / scratch
  float* nodes = nullptr;
  float* nodes_alt = nullptr;
  float* edges = nullptr;
  void* A1 = nullptr;
  float* Y = nullptr;
  float* logits = nullptr;
  int64_t chunk_cap = 0;
  float* node_out = nullptr;
  float* edge_out = nullptr;
  // block export (blocks.cu): global ids per row, packed image shift per
  // view edge, per-item value offsets (built on first export after a prepare)
  int* row_global = nullptr;
  uint32_t* eshift = nullptr;
  struct BlockState* blk = nullptr;
  bool blk_ready = false;  // blk's per-item offsets match the prepared view
  // allocated elements of the view buffers (grow)
  size_t cap_row_slot = 0, cap_src = 0, cap_dst = 0, cap_dir = 0, cap_dist = 0, cap_seg = 0, cap_nodes = 0,
         cap_nodes_alt = 0, cap_edges = 0, cap_a1 = 0, cap_y = 0, cap_logits = 0, cap_node_out = 0,
         cap_edge_out = 0, cap_send_rows = 0, cap_send_buf = 0, cap_row_global = 0, cap_eshift = 0;
  bool a1_tc_clean = false;  // A1 holds zeros in every tensor-core K padding slot
  int a1_zero_mode = 0;      // which image's padding is zero (1 bf16 tiles, 2 fp16x3 split)
  // training (train.cu): the forward saves every block's input tables when
  // save_inputs is set -- the node table after the block's halo exchange
  // (per block) and the edge table entering each layer (per layer)
  bool save_inputs = false;
  std::vector<float*> saved_nodes, saved_edges;
  TrainState* train = nullptr;
  bool train_stale = true;  // set by every prepare
  int64_t block_values = 0;
  cudaEvent_t ev[8];
  // per-exchange events of the last forward (start, lined up, done) and the
  // halo bytes it sent + received
  std::vector<cudaEvent_t> halo_ev;
  std::vector<int> halo_marks;
  int64_t halo_bytes = 0;
  // optional per-category kernel timing (esg_profile_*): events around launches
  bool profile = false;
  // esg_forward_async without timing: the host does not wait for the forward
  // (its end event is synchronised by esg_forward_wait / the next call)
  bool defer_sync = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, int>> marks;  // (category, first event index)
  double prof_ms[ESG_PROF_NCAT] = {0};
  int64_t prof_n[ESG_PROF_NCAT] = {0};
  // streamed outputs (esg_forward with pinned host buffers): heads of the
  // final tables are computed as soon as they are final and copied on copy_st
  float* host_node_out = nullptr;
  float* host_edge_out = nullptr;
  cudaStream_t copy_st = nullptr;
  std::vector<cudaEvent_t> out_ev;
  size_t out_ev_used = 0;
  // copies of a previous call may still read node_out / edge_out (async
  // forward): heads of the next forward wait on this event first
  cudaEvent_t copies_done = nullptr;
  bool copies_pending = false;
  int precision = ESG_LINEAR_FP32;
  int prefetch = 1;  // L2 prefetch mode of the rotate kernels (ESG_PREFETCH=0/1/2)
  size_t a1_elem = 4;
};

void free_ptr(void* p);
void blocks_free(DeviceModel* D);  // blocks.cu

}  // namespace esg
