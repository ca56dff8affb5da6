/*
 * vpipe_b200.h — C ABI of the B200-native vocabulary-parallel layers.
 *
 * This is the drop-in boundary for the reference's vocab-math module
 * (/root/reference/proj/include/vpipe/vocab_math.hpp, "VM.hpp" below, and
 * /root/reference/proj/src/vocab_math.cpp, "VM.cpp").  Every entry point
 * names the reference function it replaces.  The C++ mirror of the
 * reference's own header (same names, structs and argument order) is
 * include/vpipe/vocab_math.hpp, implemented on top of this ABI.
 *
 * Conventions
 *   - All tensors are DEVICE buffers owned by the caller, row-major, with
 *     explicit leading dimensions in elements.  Operands X and W are bf16;
 *     gradients, losses and stats are fp32; ids are int64.
 *   - h and every leading dimension of a bf16 tensor must be multiples of 8
 *     (16-byte TMA rows); base pointers 16-byte aligned.
 *   - Calls are asynchronous on the context's stream.  Hot calls do not
 *     allocate once vp_ctx_reserve / the first call of a shape has sized the
 *     workspace.
 *   - Return codes: VP_OK, VP_EINVAL (the reference's std::invalid_argument,
 *     same message text, retrievable with vp_last_error()), VP_ECUDA,
 *     VP_ENCCL (collective backend, NCCL or loopback).  Errors found on the
 *     device (negative token ids, VM.cpp:232, :247; labels outside [0, V),
 *     VM.cpp:18, checked by the loss, C1 and naive kernels, negative labels
 *     also by pass T) are reported by the next vp_ctx_sync() as VP_EINVAL.
 *   - Sharding: shard k owns vocab rows [row_begin, row_end) (VM.cpp:65-80).
 *     A context either drives several shards on ONE device (functions take
 *     arrays of n shard states; the reference's in-process "collectives"
 *     become device kernels, merged in k order), or — after
 *     vp_ctx_comm_init — is one rank of an NCCL group with one shard per
 *     rank (n must be 1; the exchanges are NCCL collectives over NVLink).
 */
#ifndef VPIPE_B200_H_
#define VPIPE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VP_OK 0
#define VP_EINVAL 1
#define VP_ECUDA 2
#define VP_ENCCL 3
#define VP_EINTERNAL 4

#define VP_ABI_VERSION 1

typedef struct vp_ctx_s* vp_ctx_t;
typedef struct vp_state_s* vp_state_t;

/* EmbeddingShard (VM.hpp:21-31): W_k = rows [row_begin, row_end) of W. */
typedef struct {
  const void* W;      /* bf16 [rows x h] */
  int64_t ldw;        /* elements */
  int64_t row_begin;
  int64_t row_end;
  int32_t index;      /* shard index k */
} vp_shard_t;

/* TokenBatch (VM.hpp:15-18): X [n_tok x h] plus labels [n_tok]. */
typedef struct {
  const void* X;            /* bf16 [n_tok x h] */
  int64_t ldx;
  const int64_t* labels;    /* [n_tok], global vocab ids */
  int64_t n_tok;
  int64_t h;
} vp_batch_t;

/* GlobalStats (VM.hpp:45-48): per-token global max and exp-sum, fp32 [n_tok]. */
typedef struct {
  float* m;
  float* sum;
} vp_stats_t;

/* ---- library / context ------------------------------------------------- */
int vp_abi_version(void);
const char* vp_last_error(void);

int vp_ctx_create(int device, vp_ctx_t* out);
int vp_ctx_destroy(vp_ctx_t ctx);
/* Run on an existing cudaStream_t (NULL = the legacy default stream).  A new
 * context runs on its own non-blocking stream until this is called. */
int vp_ctx_set_stream(vp_ctx_t ctx, void* stream);
void* vp_ctx_get_stream(vp_ctx_t ctx);
/* Wait for the stream; report deferred device-side argument errors. */
int vp_ctx_sync(vp_ctx_t ctx);
/* Pre-size the workspace for up to n_tok tokens, hidden h, p exchange parts. */
int vp_ctx_reserve(vp_ctx_t ctx, int64_t n_tok, int64_t h, int p);
/* Device memory plan for one rank (no GPU needed): bytes of one shard state
 * (vp_state_create: P, tile stats, A), of the context workspace at that shape
 * (after vp_ctx_reserve and the first input/output calls), and of the peer
 * buffers of the fused exchanges in a group of nranks > 1 (0 otherwise).
 * Any output pointer may be NULL.  For sizing shards and microbatches against
 * the 180 GB of HBM3e (SURVEY.md §8b "vp_workspace_query"). */
int vp_workspace_query(int64_t n_tok, int64_t h, int64_t rows, int nranks, int64_t* state_bytes,
                       int64_t* ctx_bytes, int64_t* peer_bytes);
/* Options: "cta_group" (1 or 2, default 2), "gemm_sms" (SMs used by GEMMs),
 * "raster_{logits,dx,dw}" (tile order, see GemmGeom::raster),
 * "policy_{logits,dx,dw}" (TMA L2 policy of both operands: -1 per-epilogue default,
 * 0 normal, 1 first, 2 last = the default), "policyb_{logits,dx,dw}" (B operand only;
 * logits default 1: W evict-first so X stays L2-resident),
 * "multicast" (1 = CTA-pair clusters, 2 = 4-CTA clusters sharing B by TMA multicast),
 * "nh_logits" / "nh_dx" / "nh_dw" (1 = 256x256 pair tiles, 2 = 256x512 pair tiles),
 * "force_collectives" (1 = use the NCCL group even with one rank; tests),
 * "overlap_c1" (1 = vp_run_alg2 overlaps the dX / loss all-reduce with pass T
 * on a high-priority comm stream; default 1), "comm_sms" (SMs left to NCCL
 * during the overlap and NCCL's maxCTAs; set before vp_ctx_comm_init),
 * "epi_wait" (GEMM epilogue wait: 0 try_wait loop, 1 nanosleep backoff;
 * process-wide), "store_evict_first" (1 = epilogue TMA stores with an L2
 * evict-first hint; default 0; process-wide), "store_hint_{logits,dx,dw}"
 * (per GEMM of this context: 1 evict-first, 0 normal, -1 the process-wide
 * option; default logits 1 (P), dx / dw -1),
 * "lockstep_logits" / "lockstep_dx" / "lockstep_dw" (wave lockstep of the
 * persistent GEMM's clusters every N k-blocks so co-scheduled tiles share
 * operand bands in L2; 0 = off; default 8 for all three),
 * "splits_dx" / "splits_dw" (split-K of the dX / A GEMM, whose K = V_k leaves
 * few tile waves, and of the dW GEMM for small shards: 0 = chosen from the wave
 * quantisation (default), 1 = off, 2..32 = forced; partial sums are added in
 * split order, so results are deterministic),
 * "split_workspace" (GEMMs whose tiles fill less than half a wave split K into
 * concurrent units that store partials into a context workspace, summed in
 * split order by a reduction kernel: 1 = auto (default), 0 = never (ordered
 * in-place splits only), 2 = whenever split), "split_min_kb" (ordered splits
 * keep at least this many 64-deep k-blocks per unit; default 64),
 * "cooperative" (1 = persistent GEMMs launched cooperatively, so the whole grid
 * is co-resident, which their cross-CTA waits rely on when kernels of other
 * streams hold SMs; default 1; process-wide),
 * "tma_store" (1 = GEMM epilogues store through smem staging + TMA, the
 * default; 0 = per-thread st.global; process-wide),
 * "debug_logit_scale_ppm" (fault injection for verification tools: pass-S
 * logits scaled by 1 + ppm * 1e-6; 0 = off),
 * "accumulate_grad_w" (1 = the T passes add dW_k into grad_w: gradient
 * accumulation, or tied input/output embeddings sharing the shard's buffer
 * with vp_input_backward(accumulate=1); R/PAPER.md:333),
 * "persist_logits" / "persist_dw" (1 = the logits / dW GEMM launch carries a
 * persisting L2 access-policy window over its X operand, with the device's
 * persisting L2 set-aside sized on first use: with raster_logits=32, or with
 * raster_dw=-8 policy_dw=0 policyb_dw=2, DRAM bytes per launch fall to about
 * the algorithmic bytes, but in-step throughput measured 0.5-1.5% lower
 * (profiles/r02y_*, r02z_*); default 0),
 * "peer_input" (vp_input_forward_gathered in a group: 1 = every rank writes
 * its owned rows at their token index into a peer-mapped buffer and, after a
 * one-float barrier, reads every row from its owner's buffer (NVLink P2P / CUDA
 * IPC): two kernels and no host-side sizes, so the call is capturable;
 * default 1; 0 or an unmappable group = the packed broadcasts),
 * "fused_c1" (vp_run_alg2 / vp_run_alg2_chunked / vp_run_alg1 / vp_program_run
 * in a group of nranks > 1, or a 1-rank group with "force_collectives" (alg1:
 * the dX of pass T, then C2):
 * 1 = the dX GEMM of pass S stores each A_k tile straight into the buffer of
 * the rank that owns those token rows from its epilogue, over peer memory
 * (NVLink P2P or CUDA IPC), the label rows follow, and at C1 each owner combines its rows from
 * local memory and every rank pulls the owners' rows into grad_x with its copy
 * engines — a reduce-scatter fused into the GEMM epilogue and an SM-free
 * all-gather instead of an all-reduce of [n_tok x h] fp32 partials;
 * grad_x has the bits of a one-GPU run over the same shards.  Default 1; the
 * group falls back to the all-reduce when a rank cannot map its peers.
 * 0 = always the all-reduce). */
int vp_ctx_set_option(vp_ctx_t ctx, const char* key, int64_t value);
/* The reference's per-row logit_shift test hook (VM.cpp:41-43,
 * oracle_output_layer's `logit_shift`): subsequent pass-S logits are
 * Y[i, :] + shift[i] (device fp32 [n_tok], kept by pointer; NULL clears it).
 * Softmax, loss and gradients are shift-invariant (test_vocab_math.cpp:74-84). */
int vp_ctx_set_logit_shift(vp_ctx_t ctx, const float* shift);
/* Test hook: occupy `nsms` SMs (one block per SM, all of its shared memory)
 * for `microseconds` on `stream` (NULL = legacy default stream), as NCCL's
 * kernels do during the overlapped exchanges; used to show that the
 * cooperative persistent GEMMs neither deadlock nor change results when other
 * streams hold SMs. */
int vp_debug_occupy_sms(vp_ctx_t ctx, void* stream, int nsms, int64_t microseconds);
/* Number of kernels this context has launched (evidence counter). */
int64_t vp_ctx_launch_count(vp_ctx_t ctx);
/* Number of fused C1 exchanges (option "fused_c1") this context has run;
 * -1 for a null context (evidence counter). */
int64_t vp_ctx_fused_c1_count(vp_ctx_t ctx);
/* Number of vp_input_forward_gathered / vp_input_backward_gathered calls that
 * took the peer-memory path (option "peer_input"); -1 for a null context
 * (evidence counter). */
int64_t vp_ctx_peer_input_count(vp_ctx_t ctx);
/* Per-GEMM CUDA-event timing on the launching stream.  Returns (and resets)
 * the accumulated milliseconds / launch counts per GEMM kind since the last
 * call — [0] logits+stats (K1), [1] fp32 logits (naive F1), [2] dX (K3),
 * [3] dW (K4) — then enables (enable=1) or disables timing.  Synchronises. */
int vp_ctx_gemm_timing(vp_ctx_t ctx, int enable, double* ms_out4, int64_t* count_out4);

/* Collective group of a context (one shard per rank).  Rank 0 creates an id,
 * every rank calls vp_ctx_comm_init with it (the id travels by the caller's
 * own bootstrap: torch.distributed, MPI, a file).
 *   vp_comm_unique_id    NCCL (ncclGetUniqueId): production, one rank per GPU.
 *   vp_comm_loopback_id  loopback backend: ranks may share one GPU (threads
 *                        of one process or processes of one node); device
 *                        mailboxes + a host rendezvous.  It runs every
 *                        nranks > 1 code path of the library on a single GPU.
 *                        Not capturable into CUDA graphs.  Ranks sharing a
 *                        GPU split its SMs for the persistent GEMMs.
 * vp_ctx_comm_init dispatches on the kind of id. */
int vp_comm_unique_id(void* id128);
int vp_comm_loopback_id(void* id128);
int vp_ctx_comm_init(vp_ctx_t ctx, int nranks, int rank, const void* id128);
/* One process driving n contexts (ctxs[k] becomes rank k; drive each rank
 * from its own host thread afterwards).  Distinct devices: NCCL, all ranks
 * initialised from this thread in one group (ncclCommInitAll's pattern);
 * contexts sharing a device: the loopback backend. */
int vp_comm_init_all(vp_ctx_t* ctxs, int n);
int vp_ctx_comm_info(vp_ctx_t ctx, int* nranks, int* rank);
/* "nccl", "loopback" or "none". */
const char* vp_ctx_comm_backend(vp_ctx_t ctx);

/* ---- shard state (ShardState, VM.hpp:34-43) ----------------------------- */
/* Device buffers for one shard: P = exp(Y - m_tile) in bf16 [n_tok x rows]
 * (never the fp32 logits), per-256-column tile stats, m'/sum', the label
 * logit y[i, g_i] of owned rows, A [n_tok x h] fp32 (alg2). */
int vp_state_create(vp_ctx_t ctx, int64_t n_tok, int64_t h, int64_t rows, vp_state_t* out);
/* States belong to their context: destroy them before vp_ctx_destroy. */
int vp_state_destroy(vp_state_t st);
/* m_local / sum_local (VM.hpp:36-37), device fp32 [n_tok]. */
int vp_state_local_stats(vp_state_t st, const float** m_local, const float** sum_local);
/* A = softmax'(Y) W_k (VM.hpp:40), device fp32 [n_tok x h], alg2 only. */
int vp_state_grad_terms(vp_state_t st, const float** A, int64_t* lda);

/* Copies into caller-owned device buffers (async on the context stream). */
int vp_state_copy_local_stats(vp_ctx_t ctx, vp_state_t st, float* m_out, float* sum_out);
int vp_state_copy_grad_terms(vp_ctx_t ctx, vp_state_t st, float* A_out, int64_t ldo);

/* ---- output layer ------------------------------------------------------- */
/* alg1_pass_S (VM.cpp:151-162): logits GEMM with the fused stats epilogue.
 * batch->labels (may be NULL here, as in the reference's signature) are
 * used to capture y[i, g_i] for the loss. */
int vp_alg1_pass_S(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shard, vp_state_t st);
/* alg2_pass_S (VM.cpp:181-191): alg1_pass_S + A = softmax'·W_k
 * (B = G_k·W_k is a sparse row gather done in C1). */
int vp_alg2_pass_S(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shard, vp_state_t st);
/* merge_max_sum (VM.cpp:82-101), C1 of alg1: one NCCL all-gather of the
 * [2 x n_tok] stats + a fixed-order merge; sum *= fault_scale (VM.cpp:314). */
int vp_merge_max_sum(vp_ctx_t ctx, const vp_state_t* states, int n, double fault_scale, vp_stats_t out);
/* merge_max_sum over raw device parts m/sum laid out [p x ld] (k-th part at
 * offset k*ld), merged in k order — the host API's LocalStats entry point. */
int vp_merge_stats_raw(vp_ctx_t ctx, const float* m_parts, const float* sum_parts, int p, int64_t n, int64_t ld,
                       double fault_scale, vp_stats_t out);
/* alg1_pass_T (VM.cpp:164-179): rescale + dX and dW GEMMs of this shard. */
int vp_alg1_pass_T(vp_ctx_t ctx, vp_state_t st, vp_stats_t stats, const vp_batch_t* batch,
                   const vp_shard_t* shard, float* grad_x_partial, int64_t ldgx, float* grad_w, int64_t ldgw);
/* C2 of alg1 (VM.cpp:322): grad_x = sum_k partial_k (NCCL all-reduce, or k-ordered sum). */
int vp_reduce_grad_x(vp_ctx_t ctx, float* const* partials, int n, int64_t n_tok, int64_t h, int64_t ld,
                     float* grad_x, int64_t ldgx);
/* alg2_barrier_C1 (VM.cpp:193-211; fault path :337-350): stats merge and
 * grad_x = sum_k (A_k (.) scale_k - B_k); the only barrier of alg2. */
int vp_alg2_barrier_C1(vp_ctx_t ctx, const vp_state_t* states, const vp_shard_t* shards, int n,
                       const vp_batch_t* batch, double fault_scale, vp_stats_t out, float* grad_x, int64_t ldgx);
/* alg2_pass_T (VM.cpp:213-225): dW_k = (softmax'·scale - G_k)^T X. */
int vp_alg2_pass_T(vp_ctx_t ctx, vp_state_t st, vp_stats_t stats, const vp_batch_t* batch,
                   const vp_shard_t* shard, float* grad_w, int64_t ldgw);
/* loss_i = m_i + log(sum_i) - Y[i, g_i] at the owning shard (VM.cpp:287-292). */
int vp_output_loss(vp_ctx_t ctx, const vp_state_t* states, const vp_shard_t* shards, int n, vp_stats_t stats,
                   const vp_batch_t* batch, float* loss);
/* softmax columns of one shard (assemble_forward, VM.cpp:281-286), fp32
 * [n_tok x rows] — parity/debug materialisation only. */
int vp_shard_softmax(vp_ctx_t ctx, vp_state_t st, vp_stats_t stats, float* out, int64_t ldo);
/* ShardState::Y (VM.hpp:35) on demand: fp32 logits X W_k^T [n_tok x rows]
 * (one GEMM; pass S itself never stores them).  Debug / parity only. */
int vp_shard_logits(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shard, float* out, int64_t ldo);
/* ShardState::B (VM.hpp:41) on demand: B[i, :] = W_k[g_i - row_begin, :] for
 * owned labels, else 0; fp32 [n_tok x h].  Debug / parity only. */
int vp_shard_label_rows(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shard, float* out, int64_t ldo);
/* naive_partitioned_output (VM.cpp:103-149): 3 barriers, stores and
 * re-reads fp32 logits. grad_w[k] is shard k's [rows_k x h] block. */
int vp_naive_partitioned_output(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shards,
                                const vp_state_t* states, int n, vp_stats_t out, float* loss, float* grad_x,
                                int64_t ldgx, float* const* grad_w, int64_t ldgw);
/* Drivers run_alg1 / run_alg2 (VM.cpp:303-361) minus the [n_tok x V]
 * softmax assembly (use vp_shard_softmax for that). */
int vp_run_alg1(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shards, const vp_state_t* states, int n,
                double fault_scale, vp_stats_t out, float* loss, float* grad_x, int64_t ldgx, float* const* grad_w,
                int64_t ldgw);
int vp_run_alg2(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shards, const vp_state_t* states, int n,
                double fault_scale, vp_stats_t out, float* loss, float* grad_x, int64_t ldgx, float* const* grad_w,
                int64_t ldgw);
/* Memory-bounded run_alg2 (the paper's future-work remark on
 * avoiding the softmax round trip, R/PAPER.md:498): the batch is processed as
 * consecutive chunks of at most chunk_tokens tokens (softmax rows are
 * independent), each through S -> C1 -> T with the per-chunk exchanges, so P
 * takes chunk_tokens x V_k instead of n_tok x V_k; dW accumulates over the
 * chunks.  `states` are created for min(chunk_tokens, n_tok) tokens.  Results
 * equal vp_run_alg2's to the parity tolerances (dW sums chunk partials). */
int vp_run_alg2_chunked(vp_ctx_t ctx, const vp_batch_t* batch, const vp_shard_t* shards, const vp_state_t* states,
                        int n, int64_t chunk_tokens, double fault_scale, vp_stats_t out, float* loss, float* grad_x,
                        int64_t ldgx, float* const* grad_w, int64_t ldgw);

/* ---- input layer -------------------------------------------------------- */
/* input_forward (VM.cpp:227-236): out[i] = W_k[tok_i - row_begin] if owned,
 * else 0 (accumulate=0), or out[i] += owned row (accumulate=1).  bf16. */
int vp_input_forward(vp_ctx_t ctx, const int64_t* tokens, int64_t n_tok, int64_t h, const vp_shard_t* shard,
                     void* out, int64_t ldo, int accumulate);
/* input_backward (VM.cpp:238-251): dE_k[t - row_begin] += grad_out[i] for
 * owned tokens in ascending i (deterministic sort + segmented sum); dE_k
 * zeroed first unless accumulate.  grad_out bf16 (grad_is_f32=0) or fp32. */
int vp_input_backward(vp_ctx_t ctx, const void* grad_out, int64_t ldg, int grad_is_f32, const int64_t* tokens,
                      int64_t n_tok, int64_t h, const vp_shard_t* shard, float* grad_w, int64_t ldgw,
                      int accumulate);
/* The input layer's forward over the whole group without the zero-padded
 * all-reduce: every rank gets out[i] = W[tok_i] (a zero row when no shard owns
 * tok_i), i.e. input_forward summed over the shards (VM.cpp:227-236 +
 * R/PAPER.md:582).  Default (option "peer_input"): owned rows are written at
 * their token index into peer-mapped buffers and every rank pulls each row
 * from its owner (about half the bytes of the sum all-reduce; capturable after
 * the first call).  Fallback: ranks pack the rows they own and exchange them in
 * one grouped broadcast per rank (synchronises the stream once; not
 * capturable).  Pure copies, bit-exact.  One rank: equals vp_input_forward. */
int vp_input_forward_gathered(vp_ctx_t ctx, const int64_t* tokens, int64_t n_tok, int64_t h,
                              const vp_shard_t* shard, void* out, int64_t ldo);
/* The input layer's pre-backward broadcast (R/PAPER.md:582): grad_out of the
 * embedding output [n_tok x h] (row stride ldg; fp32 or bf16), in place from
 * rank `root` to every rank of the group.  No-op without a group. */
int vp_input_grad_broadcast(vp_ctx_t ctx, void* grad_out, int64_t ldg, int grad_is_f32, int64_t n_tok, int64_t h,
                            int root);
/* The input layer's backward over the whole group: vp_input_grad_broadcast
 * from `root` followed by vp_input_backward of this rank's shard, without
 * sending every rank the whole gradient.  grad_out is read on `root` only
 * (other ranks may pass NULL).  Default (option "peer_input"): root stages
 * grad_out in a peer-mapped buffer and each rank's ordered scatter reads just
 * the rows of the tokens its shard owns over NVLink (about 1/N of the
 * gradient per rank instead of all of it); fallback: the broadcast into a
 * context buffer.  Same bits as broadcast + input_backward.  One rank: equals
 * vp_input_backward. */
int vp_input_backward_gathered(vp_ctx_t ctx, const void* grad_out, int64_t ldg, int grad_is_f32,
                               const int64_t* tokens, int64_t n_tok, int64_t h, const vp_shard_t* shard,
                               float* grad_w, int64_t ldgw, int accumulate, int root);
/* In-place sum all-reduce over the context's NCCL group (the input layer's
 * post-forward all-reduce, R/PAPER.md:582).  dtype 0 = fp32, 1 = bf16. */
int vp_allreduce_sum(vp_ctx_t ctx, void* buf, int64_t count, int dtype);

/* ---- vocabulary-pass executor (pipeline integration) --------------------- */
/* A reference DeviceProgram (P/include/vpipe/schedule.hpp:95-100) in the text
 * form of serialize_program (P/src/schedule.cpp:512-529); parse errors are
 * VP_EINVAL with the reference parser's messages (:531-577). */
typedef struct vp_program_s* vp_program_t;
int vp_program_parse(const char* text, vp_program_t* out);
int vp_program_destroy(vp_program_t prog);
/* barriers: 0 = no vocabulary passes, 1 = Algorithm 2 (vocab2), 2 = Algorithm 1
 * (vocab1, interlaced, vhalf-vocab1), method_barriers (P/src/schedule.cpp:80-88);
 * p devices, n microbatches. */
int vp_program_info(vp_program_t prog, int* barriers, int* p, int* n);
/* validate_dependencies (P/src/schedule.cpp:390-447) for the vocabulary passes
 * C0 -> S -> C1 -> T [-> C2]: violations '\n'-separated into buf (NUL-terminated,
 * truncated to buflen), their number in *count; structural errors (missing or
 * duplicate passes) as one message, in the reference's wording. */
int vp_program_validate(vp_program_t prog, char* buf, int64_t buflen, int* count);
/* Executes the program's vocabulary passes in program order (F/B/IF/IB are the
 * caller's and are skipped): S / T on the context stream, the barrier
 * exchanges of C1 (Algorithm 2) / C2 (Algorithm 1) on the high-priority comm
 * stream, overlapping the passes that follow.  NCCL group (nranks == p): this
 * rank runs device `rank` with n_shards = 1; local: every device on this GPU,
 * n_shards = p.  batches, stats, loss, grad_x: one per microbatch (n);
 * states: [n_shards x n] shard-major; grad_w: one per shard, zeroed, then dW
 * of every microbatch accumulates into it.  C0 broadcasts X_i from device p-1
 * (NCCL group: X_i of the other ranks is overwritten). */
int vp_program_run(vp_ctx_t ctx, vp_program_t prog, const vp_batch_t* batches, const vp_shard_t* shards,
                   int n_shards, const vp_state_t* states, vp_stats_t* stats, float* const* loss,
                   float* const* grad_x, int64_t ldgx, float* const* grad_w, int64_t ldgw);

/* ---- CUDA graphs ----------------------------------------------------------- */
/* Capture the context's work (any vp_* calls on it, including the comm-stream
 * fork/join and NCCL calls) into a graph replayed with one launch.  Workspace
 * buffers must already be sized (run the same calls once eagerly first);
 * GEMM timing must be off. */
typedef struct vp_graph_s* vp_graph_t;
int vp_ctx_capture_begin(vp_ctx_t ctx);
int vp_ctx_capture_end(vp_ctx_t ctx, vp_graph_t* out);
int vp_graph_launch(vp_graph_t graph, vp_ctx_t ctx);
int vp_graph_destroy(vp_graph_t graph);

#ifdef __cplusplus
}
#endif
#endif /* VPIPE_B200_H_ */
