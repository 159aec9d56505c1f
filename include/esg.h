/* esg.h -- C ABI of the B200-native esgnn hot path (libesg_b200.so).
 *
 * Drop-in boundary for the reference's C++20 library API (no FFI exists in
 * the reference; these are the entry points its façade would bind).  Every
 * function returns an ESG_* status; esg_last_error() gives the message.  The
 * C++ façade in paper_2507_03840_b200/csrc/esgnn_b200.hpp rethrows the
 * matching esgnn::Error subclass (core/error.h:11-51), mirroring the CLI's
 * exit-code mapping usage->2, data->3, divergence->4 (esgnn_main.cpp:221-233).
 *
 * Conventions: host arrays are caller-owned; device buffers are owned by the
 * context / handle that created them.  A context drives one GPU and is not
 * thread-safe (one host thread or process per context, like one rank of the
 * reference's DistributedRunner).  Collectives are issued in the same order
 * on every rank (transport.h:17-20 lockstep contract).
 */
#ifndef ESG_H_
#define ESG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ESG_OK = 0,
  ESG_ERR_OTHER = 1,
  ESG_ERR_USAGE = 2,      /* esgnn::UsageError */
  ESG_ERR_DATA = 3,       /* esgnn::DataError / ShapeError / ParseError */
  ESG_ERR_DIVERGENCE = 4, /* esgnn::DivergenceError */
  ESG_ERR_NCCL = 5,       /* esgnn::TransportError */
  ESG_ERR_CUDA = 6,
  ESG_ERR_OOM = 7
};

/* precision of the SO(2) linears (everything else is fp32 state with fp64
 * geometry): FP32 = fp32-faithful products on the tensor cores -- tcgen05
 * kind::f16 over a 3-term fp16 split with power-of-two scales (l_max 4,
 * e_width 16; so2_f16x3.cu) or kind::tf32 over a 3xTF32 split (other shapes
 * and the training reverse pass), within the fp32 tolerance of the float
 * oracle; BF16 = tcgen05 kind::f16 on bf16 operands with fp32 accumulation
 * in TMEM (throughput mode). */
enum { ESG_LINEAR_FP32 = 0, ESG_LINEAR_BF16 = 1 };

typedef struct esg_ctx esg_ctx;
typedef struct esg_graph esg_graph;
typedef struct esg_plan esg_plan;
typedef struct esg_model esg_model;

typedef struct esg_timing {
  double forward_ms;      /* first init kernel -> last head kernel (CUDA events) */
  double message_ms;      /* message passing only (all 2*M blocks) */
  double halo_ms;         /* sum over the 2*M exchanges: start -> last recv, rank skew included */
  double heads_ms;
  int64_t exchanges;      /* exactly 2*M per forward (acceptance.cpp:298) */
  int64_t gpu_launches;   /* kernels this library launched in the call */
  /* with esg_profile on, a one-float allreduce lines the ranks up before each
   * exchange: halo_skew_ms is the waiting for the slowest rank, and
   * halo_exchange_ms pack start -> last recv after it (otherwise -1 and
   * halo_ms); halo_bytes: the bytes this rank sent plus received */
  double halo_skew_ms;
  double halo_exchange_ms;
  int64_t halo_bytes;
} esg_timing;

const char* esg_last_error(void);
int esg_version(void);

/* ---- context (one GPU, optional NCCL communicator) ------------------- */
int esg_nccl_unique_id_size(void);
int esg_nccl_get_unique_id(void* out /* esg_nccl_unique_id_size() bytes */);
/* world > 1 requires nccl_id (the same bytes on every rank). */
int esg_ctx_create(int device, int rank, int world, const void* nccl_id, esg_ctx** out);
int esg_ctx_destroy(esg_ctx* ctx);
int esg_ctx_synchronize(esg_ctx* ctx);

/* ---- structures (structure.h:12-36, synthetic.h:17-41) ---------------- */
/* AtomicStructure::wrap (structure.cpp:26-38), host. */
int esg_wrap_positions(int n_atoms, double* pos /* n*3, in place */, const double cell[9],
                       const uint8_t pbc[3]);
/* model::make_jittered_lattice (synthetic.cpp:17-41), host input generator. */
int esg_jittered_lattice(int n_atoms, double spacing, double jitter, int n_cycle, const int* cycle,
                         uint64_t seed, double* pos_out, double cell_out[9], int* species_out);
/* structures::read_extxyz_file (extxyz.h:17, extxyz.cpp:62-126): atom count,
 * Cartesian positions (n*3), atomic numbers, cell rows (Lattice; the
 * identity when absent, as AtomicStructure's default) and pbc.  Pass pos / species / cell / pbc NULL to get the count
 * only.  Malformed files: ESG_ERR_DATA with the line number (ParseError,
 * core/error.h:27-35). */
int esg_extxyz_read(const char* path, int64_t* n_atoms, double* pos, int32_t* species, double cell[9],
                    uint8_t pbc[3]);
/* structures::write_extxyz_file (extxyz.h:20, extxyz.cpp:128-151): the same
 * text, %.17g numbers (exact round trip). */
int esg_extxyz_write(const char* path, int64_t n_atoms, const double* pos, const int32_t* species,
                     const double cell[9], const uint8_t pbc[3]);
/* structures::tile (structure.cpp:40-63), host. */
int esg_tile(int n_atoms, const double* pos, const double cell[9], const uint8_t pbc[3],
             const int* species, const int reps[3], double* pos_out, double cell_out[9],
             int* species_out);

/* ---- graph: structures::build_graph (graph.h:37, graph.cpp:55-131) ---- */
/* Builds the periodic cutoff graph on the GPU: a destination-major CSR
 * whose edges are ordered by (dst, src, shift) exactly like Graph::edges. */
int esg_build_graph(esg_ctx* ctx, int n_atoms, const double* pos, const double cell[9],
                    const uint8_t pbc[3], double r_cut, esg_graph** out);
int esg_graph_destroy(esg_graph* g);
int esg_graph_info(const esg_graph* g, int* n_nodes, int64_t* n_edges);
/* Copies Graph::edges to host SoA arrays (any pointer may be NULL). */
int esg_graph_export(const esg_graph* g, int32_t* src, int32_t* dst, int32_t* shift /* E*3 */,
                     double* disp /* E*3 */, double* dist);
/* Graph::in_degrees (graph.cpp:49-53) and incoming_ranges offsets (N+1). */
int esg_graph_in_degrees(const esg_graph* g, int32_t* deg);
int esg_graph_offsets(const esg_graph* g, int64_t* dst_off /* N+1 */);

/* ---- partition::lownn_partition (partition.h:24, lownn.cpp:105-133) --- */
/* pos are the UNWRAPPED input positions (model_run.cpp:68 passes in.s). */
int esg_lownn_partition(int n_atoms, const double* pos, const double cell[9], const uint8_t pbc[3],
                        const int32_t* in_degree, int depth, double r_cut, int32_t* node_to_part);
/* The same assignment computed on the device of `ctx`: one
 * pass per bisection level, segmented radix sorts by (coordinate, atom id),
 * a weight scan and a per-segment first-minimiser split.  Host in / out. */
int esg_lownn_partition_gpu(esg_ctx* ctx, int n_atoms, const double* pos, const double cell[9], const uint8_t pbc[3],
                            const int32_t* in_degree, int depth, double r_cut, int32_t* node_to_part);

/* ---- partition metrics (partition.h:31-62, metrics.cpp:49-166)
 * compute_metrics on the device from the graph CSR and an assignment
 * (n_parts <= 4096).  parts (n_parts entries) and volume (n_parts x n_parts,
 * volume[from * n_parts + to] = distinct source nodes part `from` packs for
 * part `to` per exchange, write_dot's edge weights) may be NULL. */
typedef struct esg_part_stats {
  int64_t nodes, edges, recv_volume; /* PartStats (partition.h:31-36) */
  int32_t neighbors, pad;
} esg_part_stats;
typedef struct esg_metrics {
  double node_imbalance, edge_imbalance, mean_neighbors; /* Metrics (partition.h:38-46) */
  int64_t total_recv, cut_edges;
  int32_t max_neighbors, n_parts;
} esg_metrics;
int esg_partition_metrics(const esg_graph* g, const int32_t* node_to_part, int n_parts, esg_metrics* m,
                          esg_part_stats* parts, int64_t* volume);
/* metrics_json (nlohmann dump(2) format) and write_dot text; *len receives
 * the text length, out (capacity cap, NUL-terminated) may be NULL to size. */
int esg_metrics_json(const esg_metrics* m, const esg_part_stats* parts, char* out, int64_t cap, int64_t* len);
int esg_partition_dot(const int64_t* volume, const esg_part_stats* parts, int n_parts, char* out, int64_t cap,
                      int64_t* len);
/* write_assignment_file / read_assignment_file ("node part" lines). */
int esg_assignment_write(const char* path, const int32_t* node_to_part, int64_t n);
int esg_assignment_read(const char* path, int32_t* node_to_part, int64_t cap, int64_t* n, int* n_parts);

/* ---- runtime::build_comm_plan (comm_plan.h:35, comm_plan.cpp:11-106) -- */
int esg_plan_build(const esg_graph* g, const int32_t* species, const int32_t* node_to_part,
                   int n_parts, int rank, esg_plan** out);
/* Same plan from host CSR arrays (dst_off[N+1], src[E]); needs no GPU. */
int esg_plan_build_host(int n_nodes, const int64_t* dst_off, const int32_t* src, const int32_t* species,
                        const int32_t* node_to_part, int n_parts, int rank, esg_plan** out);
int esg_plan_destroy(esg_plan* p);
/* info[0..4] = n_rows, n_owned, n_edges, n_neighbors, total_send_rows */
int esg_plan_info(const esg_plan* p, int64_t info[5]);
/* Any pointer may be NULL.  edge_index maps view edges to global edges. */
int esg_plan_export(const esg_plan* p, int32_t* row_global, int32_t* row_species,
                    int32_t* edge_index, int32_t* src_row, int32_t* dst_row, int32_t* nbr_peer,
                    int32_t* nbr_recv_row, int32_t* nbr_recv_count, int32_t* nbr_send_count,
                    int32_t* send_rows /* concatenated in neighbour order */);

/* ---- harmonics::coupling_matrix (clebsch_gordan.h:19) ------------------ */
/* (2L+1) x ((2la+1)(2lb+1)) row-major real-basis coupling block, host. */
int esg_coupling_matrix(int la, int lb, int L, double* out);

/* ---- model::Network<float> (network.h:77-228) ------------------------- */
typedef struct esg_model_config {
  int l_max, e_width, layers, n_radial; /* ModelConfig (network.h:16-35) */
  double r_cut;
  uint64_t seed;
  int gate_enabled;
  int linear_precision; /* ESG_LINEAR_* */
} esg_model_config;

/* basis: species Z ascending or not; shells concatenated per species.  ctx
 * may be NULL for a host-only model (parameter registration / init / hash). */
int esg_model_create(esg_ctx* ctx, const esg_model_config* cfg, int n_species, const int* z,
                     const int* n_shells, const int* shells, esg_model** out);
int esg_model_destroy(esg_model* m);
int esg_model_set_precision(esg_model* m, int linear_precision);
/* ParamStore (params.h:40-107): entries in registration order. */
int esg_model_init_params(esg_model* m); /* ParamStore::init(seed) */
int64_t esg_model_param_count(const esg_model* m);
int esg_model_n_entries(const esg_model* m);
int esg_model_entry(const esg_model* m, int i, const char** name, int* rows, int* cols,
                    int64_t* offset);
int esg_model_get_params(const esg_model* m, float* out);
int esg_model_set_params(esg_model* m, const float* in); /* uploads + repacks */
uint64_t esg_model_param_hash(const esg_model* m); /* ParamStore::value_hash */
int esg_model_out_len(const esg_model* m);           /* HeadLayout::out_len */

/* Network::prepare (network.h:98-105) on a rank view: plan may be NULL for the
 * serial view of g (serial_view, graph_view.h:37-56). */
int esg_prepare(esg_model* m, const esg_graph* g, const esg_plan* plan, const int32_t* species);
int esg_prepared_info(const esg_model* m, int64_t info[3]); /* n_rows, n_owned, n_edges */

/* DistributedRunner::forward + heads (distributed.h:193, network.h:115-164).
 * Host outputs may be NULL (results stay on the device).  When the given
 * host buffers are pinned (cudaHostAlloc / cudaHostRegister), the heads of
 * each final chunk are computed and copied while the last edge block still
 * runs; pageable buffers are filled after the forward.  Same values either way. */
int esg_forward(esg_model* m, float* node_out /* n_owned*out_len */,
                float* edge_out /* n_edges*out_len */, esg_timing* timing);
/* The same with pinned host buffers, returning once the compute is done and
 * the output copies are queued; esg_forward_wait completes them (the buffers
 * must not be read or reused before).  A following forward runs while those
 * copies drain and waits for them only before its heads overwrite the device
 * outputs.  With timing == NULL (and profiling off) the call returns as soon
 * as the forward is queued -- the host can build the next structure's graph
 * meanwhile -- and esg_forward_wait also waits for the forward.  Pageable
 * buffers: identical to esg_forward. */
int esg_forward_async(esg_model* m, float* node_out, float* edge_out, esg_timing* timing);
int esg_forward_wait(esg_model* m);
/* Per-category kernel timing with CUDA events on the launching stream.
 * esg_profile(m, enable, ms, counts): copies the accumulated milliseconds
 * and launch counts (ESG_PROF_NCAT entries each, may be NULL), then if
 * enable >= 0 resets the accumulators and switches profiling on/off. */
enum {
  ESG_PROF_INIT = 0,
  ESG_PROF_ROTATE_IN = 1,
  ESG_PROF_SO2 = 2,
  ESG_PROF_ROTATE_OUT = 3,
  ESG_PROF_NODE = 4,
  ESG_PROF_HEADS = 5,
  ESG_PROF_HALO = 6,
  ESG_PROF_COPY = 7,
  ESG_PROF_NCAT = 8
};
int esg_profile(esg_model* m, int enable, double* ms, int64_t* counts);

/* Device pointers of the last forward's outputs / features (valid until the
 * next forward or destroy). */
int esg_forward_outputs(const esg_model* m, const float** node_out, const float** edge_out,
                        const float** node_features, const float** edge_features);
/* Rows [first, first + count) of the last forward's node / edge head outputs
 * (out_len floats each) to host; either pointer may be NULL. */
int esg_outputs_export(const esg_model* m, int64_t node_first, int64_t node_count, float* node_out,
                       int64_t edge_first, int64_t edge_count, float* edge_out);
/* Node / edge feature tables (n_rows*H*E / n_edges*H*E) to host. */
int esg_features_export(const esg_model* m, float* nodes, float* edges);

/* Per-edge rotation blocks, kernels.h:43-68 build_edge_rotations (align_to_y,
 * align.cpp:32-39, then wigner_blocks, wigner.cpp:47-83) on the device: the
 * fp64 displacements (host, E*3) are rounded to fp32 as Network::prepare's
 * view does and the same in-register recursion the message kernels use
 * fills blocks (host, E * sum_l (2l+1)^2 floats: D_0..D_lmax row-major,
 * EdgeRotations' stride).  l_max 1..6. */
int esg_edge_rotations(esg_ctx* ctx, int64_t n_edges, const double* disp, int l_max, float* blocks);

/* ---- block export ------------------------
 * The blocks of the last forward, replacing Network::assemble_blocks
 * (network.h:168-184), blocks_to_uncoupled (block_matrix.cpp:66-88) and the
 * text gather to rank 0 (model_run.cpp:103-120).  Items are this rank's
 * owned atoms (key (g, g, 0)) then its owned edges in global edge order
 * (key (src, dst, shift)); each block is n_orb(Z_i) x n_orb(Z_j), row-major,
 * values concatenated in item order.  basis: ESG_BLOCKS_COUPLED (fill_block:
 * head segments placed per shell-pair rectangle) or ESG_BLOCKS_UNCOUPLED
 * (to_block per shell pair); symmetrize_onsite (uncoupled only) replaces
 * (i, i, 0) blocks by 0.5 (B + B^T) (blocks_to_uncoupled's flag). */
#define ESG_BLOCKS_COUPLED 0
#define ESG_BLOCKS_UNCOUPLED 1
typedef struct esg_block_key {
  int32_t i, j, ix, iy, iz; /* BlockKey (block_matrix.h:21-25) */
  uint16_t rows, cols;
} esg_block_key; /* 24 bytes; the shard's key record */
int esg_blocks_count(esg_model* m, int64_t* n_blocks, int64_t* n_values);
/* Keys and fp64 values to host memory (either may be NULL). */
int esg_blocks_export(esg_model* m, int basis, int symmetrize_onsite, esg_block_key* keys, double* values);
/* The same into device memory (value_bytes 8: fp64, 4: fp32), one launch
 * each; kernel_ms (may be NULL) receives their device time. */
int esg_blocks_export_device(esg_model* m, int basis, int symmetrize_onsite, int value_bytes, void* d_keys,
                             void* d_values, float* kernel_ms);
/* This rank's shard file (flat block-sparse binary, layout in DESIGN.md §3
 * and csrc/blocks_io.h), streamed through pinned staging buffers. */
int esg_blocks_write_shard(esg_model* m, const char* path, int basis, int symmetrize_onsite, int value_bytes);
/* block_matrix.cpp:90-101 write_blocks of this rank's blocks (BlockKey
 * order, 17 significant digits): for one rank, model_run's
 * blocks_coupled.txt / blocks_uncoupled.txt.  Small configurations. */
int esg_blocks_write_text(esg_model* m, const char* path, int basis, int symmetrize_onsite);
/* block_matrix.cpp:109-128 read_blocks_file (e.g. training targets): pass
 * keys / values NULL to get the sizes; blocks in BlockKey order; parse errors
 * are ESG_ERR_DATA with the line number. */
int esg_blocks_read_text(const char* path, int64_t* n_blocks, int64_t* n_values, esg_block_key* keys,
                         double* values);
/* Rank 0's gathered text file from the ranks' shards (no device needed). */
int esg_blocks_merge_text(const char* const* shard_paths, int n_shards, const char* out_path);
/* Network::build_targets (network.h:187-214): head-space targets and masks of
 * the prepared view (n_owned x out_len, n_edges x out_len, view order) from
 * uncoupled target blocks (keys + row-major values concatenated, e.g. from a
 * text file).  Items without a block keep mask 0; *count receives the number
 * of active entries (TargetBuffers::local_count).  The result feeds
 * esg_set_targets. */
int esg_build_targets(esg_model* m, int64_t n_blocks, const esg_block_key* keys, const double* values,
                      float* node_target, uint8_t* node_mask, float* edge_target, uint8_t* edge_mask,
                      int64_t* count);
/* Legacy pair: uncoupled values only, n_values from esg_blocks_count. */
int esg_blocks_size(esg_model* m, int64_t* n_values);
int esg_blocks_uncoupled(esg_model* m, double* out);

/* ---- training (config 5) -------------------------- */
/* Loss targets in head space for the prepared view (network.h:187-214
 * build_targets): node rows n_owned x out_len, edge rows n_edges x out_len in
 * view order, 1-byte masks (1 = the element is a target). */
int esg_set_targets(esg_model* m, const float* node_target, const uint8_t* node_mask, const float* edge_target,
                    const uint8_t* edge_mask);
/* Masked L1+L2 loss and parameter gradients at the current parameters
 * (distributed.h:208-226 without the optimizer step): forward on the fp32
 * path keeping every block's inputs, loss = (sum_abs + sum_sq) / n_total
 * over all ranks (ops.h:347-371, network.h:218-227), the reverse pass
 * (ops.h backward closures, kernels.h:163-250, halo backward
 * distributed.h:98-129), gradients summed over ranks in rank order in fp64
 * (allreduce_gradients, distributed.h:147-163).  partials: this rank's
 * {sum_abs, sum_sq, count}; grads: param_count floats, flat parameter
 * layout (may be NULL). */
int esg_loss_grad(esg_model* m, int64_t n_total, double partials[3], double* loss, float* grads);
/* Adam with reduce-on-plateau (optimizer.h:15-80), moments in fp64, host. */
typedef struct esg_adam_config {
  double lr, beta1, beta2, eps;
  int patience;
  double factor, threshold, min_lr;
} esg_adam_config;
void esg_adam_default_config(esg_adam_config* cfg); /* OptimizerConfig defaults */
typedef struct esg_adam esg_adam;
int esg_adam_create(const esg_model* m, const esg_adam_config* cfg, esg_adam** out);
void esg_adam_destroy(esg_adam* a);
double esg_adam_lr(const esg_adam* a);
/* DistributedRunner::train_step (distributed.h:208-235): parameter-sync
 * check (hash allgather; divergence -> status 4), loss + gradients, Adam
 * step, check again.  timing may be NULL; forward_ms = the forward,
 * message_ms = the backward (CUDA events). */
/* Optimizer::step (optimizer.h:42-72) with caller-supplied gradients: the
 * fp64-moment Adam update plus reduce-on-plateau on loss, then the parameter
 * upload when the model has a device.  esg_train_step is esg_loss_grad
 * followed by this. */
int esg_adam_apply(esg_adam* opt, esg_model* m, const float* grads, double loss);
int esg_train_step(esg_model* m, esg_adam* opt, int64_t n_total, double* loss, esg_timing* timing);

/* ---- checkpoints (checkpoint.h:15-92 + the optimizer state) --
 * The file is the reference's version-1 container (magic ESGNNCK1, config
 * text, scalar width 4, named arrays with shapes), so model::load_checkpoint
 * reads the parameters unchanged.  When opt is given an optimizer section
 * follows the arrays (magic ESGADAM1: step, lr, best, stale counter, config,
 * then the fp64 moments m and v), which the reference loader never reads and
 * esg_checkpoint_load restores for an exact resume. */
int esg_checkpoint_save(const esg_model* m, const esg_adam* opt, const char* config_text, const char* path);
/* Loads parameters (uploaded to the device when the model has one) and, if
 * opt is given, the optimizer section (status 3 if the file has none).
 * config_out (capacity cap bytes, may be NULL) receives the config text. */
int esg_checkpoint_load(esg_model* m, esg_adam* opt, const char* path, char* config_out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* ESG_H_ */
