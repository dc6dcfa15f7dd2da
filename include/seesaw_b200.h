/*
 * libseesaw_b200 — C ABI of the B200-native Seesaw re-sharding hot path.
 *
 * The reference (shardsim, /root/reference/pkg) has no native code: every op
 * below replaces an ANALYTIC cost term or transfer charge of the reference
 * with the real sm_100a kernel.  Each declaration cites the reference
 * interface it replaces (paths relative to /root/reference/pkg/src/shardsim).
 *
 * Conventions:
 *  - every pointer is caller-owned device memory unless stated; no
 *    allocation inside calls;
 *  - every call takes a cudaStream_t (as void*), is stream-ordered and
 *    asynchronous;
 *  - return 0 = OK, >0 = cudaError_t, <0 = argument error (SSB_E*); the text
 *    of the last error of the calling host thread is ssb_last_error();
 *  - all tensors are bf16 unless stated; "elements" strides are in elements.
 */
#ifndef SEESAW_B200_H_
#define SEESAW_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSB_ABI_VERSION 1

/* error codes (negative) */
#define SSB_EARG (-1)
#define SSB_EALIGN (-2)
#define SSB_EUNSUPPORTED (-3)

/* GEMM epilogues */
#define SSB_EPI_NONE 0     /* C = A.B^T                                       */
#define SSB_EPI_RESIDUAL 1 /* C = A.B^T + R (R may alias C)                   */
#define SSB_EPI_SILU_MUL 2 /* accumulator columns are (32 gate, 32 up) pairs;
                              C[:, j] = silu(gate_j) * up_j, N/2 columns     */
#define SSB_EPI_F32 3      /* C = A.B^T stored as fp32 (logits)               */
#define SSB_EPI_ROPE_KV 4  /* QKV projection + RoPE + paged KV append; only
                              through ssb_gemm_qkv_rope_kv                     */
#define SSB_EPI_ARGMAX 5   /* per-row (max, argmax) keys; only through
                              ssb_gemm_lm_head_argmax                         */

const char* ssb_last_error(void);
int ssb_version(void);
int ssb_device_sm_count(void);
/* Programmatic dependent launch of the library's GEMM / decode-attention
 * launches on (1) or off (0); returns the previous setting.  Default: the
 * SSB_PDL environment variable, else on.  Virtual ranks that share one GPU
 * and meet in the fused TP combine's device barrier must turn it off (a
 * rank's early-resident GEMM could hold the SMs its peer's producer needs). */
int ssb_set_pdl(int on);

/* CUDA IPC peer mapping for the peer-memory kernels (fused TP combine, peer
 * argmax, p2p KV re-shard): export names the cudaMalloc allocation holding
 * `ptr` (64-byte cudaIpcMemHandle_t) and ptr's offset in it; open maps a peer
 * process's handle in THIS process's context of `device` -- the GPU whose kernels will
 * dereference the pointer -- with peer access enabled on open; close it when
 * the buffer it maps is released.  (Mapping it under the exporter's device
 * instead would leave the local GPU without peer access to it.)
 * Boundary for the reference's ReshardPlan transfers, reshard.py:125-201. */
/* Debug only: CTA 0 of the next prefill attention pair-kernel launches
 * writes its per-role timeline (5 x 4096 u64: globaltimer << 24 | event << 16
 * | item << 8 | key tile) into buf; null turns it off.  tools/attn_trace.py. */
int ssb_debug_attn_trace(void* buf);
/* Debug only: stream `bytes` from src through shared memory with bulk copies
 * (ctas_per_sm x #SMs CTAs, chunk-byte pieces, a stages-deep ring), reading
 * nothing back -- the HBM read ceiling for a TMA-fed kernel. */
int ssb_debug_read_stream(const void* src, int64_t bytes, int ctas_per_sm, int chunk, int stages, void* stream);

int ssb_ipc_export(const void* ptr, void* handle_out /* 64 bytes */, int64_t* offset_out);
int ssb_ipc_open(const void* handle, int device, void** out_ptr);
int ssb_ipc_close(void* ptr, int device);

/* ------------------------------------------------------------------------
 * Dense projections (bf16 tcgen05/TMEM GEMM fed by TMA).
 * Replaces perf.py:59-65 (linear weight traffic) and perf.py:92-111 (linear
 * compute) in _quantum (sim.py:335-341).
 * C[M,N] = A[M,K] . B[N,K]^T with A, B K-major.  block_n = 0 picks the tile.
 * ---------------------------------------------------------------------- */
int ssb_gemm_bf16(const void* A, const void* B, void* C, const void* R, int M, int N, int K,
                  int lda, int ldb, int ldc, int ldr, int epilogue, int block_n, int max_ctas,
                  void* stream);
/* max_ctas > 0 caps the persistent grid (leaves SMs to a concurrent kernel,
 * e.g. decode attention of the other half-batch); 0 = one CTA per SM.
 * block_n bits 0-15: N tile (0 = auto: 128/192/224/256 by wave efficiency);
 * OR in SSB_GEMM_MC2 for CTA pairs that share the B tile by TMA multicast
 * (default single CTAs, SSB_GEMM_MC1). */
#define SSB_GEMM_MC1 (1 << 16)
#define SSB_GEMM_MC2 (1 << 17)
/* CTA pair issuing cta_group::2 MMAs (M = 256 per pair, B split across the
 * pair's shared memory). */
#define SSB_GEMM_2SM (1 << 18)
/* block_n bits 20-27: force split-K into n k-ranges (needs a workspace). */
#define SSB_GEMM_SPLIT_SHIFT 20
#define SSB_GEMM_SPLIT(n) ((n) << SSB_GEMM_SPLIT_SHIFT)
/* With SSB_GEMM_SPLIT(n): split only the tiles of the last, partial wave of
 * the persistent schedule ("tail split"); full waves run whole tiles. */
#define SSB_GEMM_TAIL (1 << 28)
/* Stream-K: whole tiles while two or more rounds remain, then the last
 * rounds' k-blocks split evenly over the persistent CTAs; shared tiles are
 * reduced in k order by their last contributor (needs a workspace). */
#define SSB_GEMM_STREAMK (1 << 29)

/* The same GEMM with a split-K workspace.  With block_n = 0 the library picks
 * (CTA pairs or single CTAs, N tile, number of k-splits) from a cost model of
 * the persistent schedule on this GPU's SM count; it only splits K when the
 * fp32 partials fit `workspace_bytes`.  Split tiles are reduced inside the
 * kernel by the last-arriving warp of each tile quadrant, summing the
 * partials in split order (deterministic).  The workspace (256-byte aligned
 * device memory) starts with a fixed 64 KiB area of tile counters (so at most
 * 4096 output tiles split) followed by the fp32 partials; it must be ZEROED
 * once before its first use, and every launch leaves the counter area zero
 * again, whatever GEMMs of whatever shapes share it.  One workspace per
 * stream: concurrent GEMMs must not share it.  This is what lets the skinny decode projections
 * (M = batch <= 512 rows, TP-sharded N or K) fill all 148 SMs. */
int ssb_gemm_bf16_ws(const void* A, const void* B, void* C, const void* R, int M, int N, int K,
                     int lda, int ldb, int ldc, int ldr, int epilogue, int block_n, int max_ctas,
                     void* workspace, int64_t workspace_bytes, void* stream);

/* RMSNorm folded into the GEMMs around it (single-GPU / TP=1 layout):
 * rmsnorm(x) * gamma @ W^T == diag(1/rms(x)) * (x @ (W * gamma)^T), so with
 * the gain folded into the consumer's weights (W[n, k] *= gamma[k]) the
 * consumer GEMM takes the residual stream x itself as A and scales its
 * accumulator rows by 1/rms in the epilogue, and the producer of x (the
 * residual-epilogue GEMM) emits the row sums of squares on the fly: no
 * rmsnorm launch, no h round trip through HBM.
 *   ss_out  (SSB_EPI_RESIDUAL only) fp32 [M][ss_parts]: sum of squares of the
 *           stored bf16 row segment of every N tile; the call writes the
 *           tile count it used into ss_parts (host side, before returning)
 *   ss_in   fp32 [M][ss_in_parts] (a producer's ss_out): every epilogue
 *           scales row m by 1/sqrt(sum_j ss_in[m][j] / hidden + eps) first
 * Either pointer may be NULL.  */
typedef struct ssb_rownorm {
  float* ss_out;
  const float* ss_in;
  int ss_in_parts;
  int hidden;
  float eps;
  int ss_parts; /* out */
} ssb_rownorm;
int ssb_gemm_bf16_rn(const void* A, const void* B, void* C, const void* R, int M, int N, int K,
                     int lda, int ldb, int ldc, int ldr, int epilogue, int block_n, int max_ctas,
                     void* workspace, int64_t workspace_bytes, ssb_rownorm* rn, void* stream);
/* The configuration block_n = 0 would pick: out_plan[3] = {mode (0 single
 * CTA, 2 CTA pair), N tile, splits (negative: tail split)}; returns the workspace bytes it needs
 * (0 without split-K), <0 on argument error. */
int64_t ssb_gemm_plan(int M, int N, int K, int epilogue, int max_ctas, int64_t workspace_bytes,
                      int32_t* out_plan);

/* ------------------------------------------------------------------------
 * KV re-shard between two parallelism layouts of the paged pool.
 * Replaces kv_reshard_route (reshard.py:170-188) / _kv_shards
 * (reshard.py:151-167), which the reference only charges as host-link bytes
 * (sim.py:382, sim.py:436-488).
 *
 * Pool of one GPU: [num_blocks][n_layers][2 (K,V)][n_heads][block_size][head_dim].
 * For a chunk of `n_ids` block ids and a list of `n_peers` peers, peer p
 * exchanges the rectangle layers [l0[p], l0[p]+nl[p]) x heads
 * [h0[p], h0[p]+nh[p]) (LOCAL indices of this GPU's pool).  The staging
 * buffer holds, peer after peer at byte offset off[p], the rectangle of every
 * block in chunk order: [n_ids][nl][2][nh][block_size][head_dim].
 * pack: pool -> staging; unpack: staging -> pool.  Peer tables live in host
 * memory (<= SSB_MAX_PEERS entries); block ids are a device int32 array.
 * ---------------------------------------------------------------------- */
#define SSB_MAX_PEERS 64
typedef struct ssb_kv_geometry {
  int n_layers;   /* local layers in the pool      */
  int n_heads;    /* local KV heads in the pool    */
  int block_size; /* tokens per block              */
  int head_dim;   /* elements per head             */
} ssb_kv_geometry;

/* QKV projection fused with RoPE and the paged KV append (one launch
 * instead of ssb_gemm_bf16 + ssb_rope_kv_append; same result bit for bit):
 * qkv[M, (nq+2nk)*head_dim] = A[M,K] . B^T, then q and k heads rotated
 * (rotate-half, fp32 tables cos/sin[max_pos][head_dim/2]) at positions[m],
 * and k, v heads of row m written to pool slot slots[m] of local layer
 * `layer` (slots may be NULL: no append; a negative slot skips the row).
 * head_dim must be 128.   Replaces the same reference terms as ssb_gemm_bf16
 * plus the KV write the cost model folds into perf.py:68-86. */
int ssb_gemm_qkv_rope_kv(const void* A, const void* B, void* qkv, int M, int K, int lda, int ldb, int ldc,
                         int nq, int nk, int head_dim, const int32_t* positions, const float* rope_cos,
                         const float* rope_sin, int max_pos, void* pool, ssb_kv_geometry geo,
                         int layer, const int64_t* slots, int block_n, int max_ctas, void* workspace,
                         int64_t workspace_bytes, ssb_rownorm* rn, void* stream);

int ssb_kv_reshard_pack(const void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                        int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                        const int32_t* nh, const int64_t* off_bytes, void* staging, void* stream);
int ssb_kv_reshard_unpack(void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                          int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                          const int32_t* nh, const int64_t* off_bytes, const void* staging,
                          void* stream);

/* Fused pack + transfer over peer memory: the same per-peer rectangles as
 * ssb_kv_reshard_pack, but peer p's rectangle is stored straight to the
 * device address dst_addr[p] (+ its position in the chunk) -- the peer's
 * receive buffer mapped into this process over NVLink (CUDA IPC) -- so the
 * copy into a send staging buffer and the separate all-to-all disappear.
 * The caller orders the kernel against the peers' use of their buffers
 * (barrier before: peers finished unpacking the previous chunk; barrier
 * after: every peer's stores landed) and then runs ssb_kv_reshard_unpack on
 * its own receive buffer. */
int ssb_kv_reshard_pack_p2p(const void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                            int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                            const int32_t* nh, const int64_t* dst_addr, void* stream);

/* ------------------------------------------------------------------------
 * Batched 2-D strided byte copy: weight column/row re-partition
 * (replaces weight_reload_plan, reshard.py:125-148, charged at
 * sim.py:328-333) and host-tier gathers.  `descs` is a DEVICE array of
 * n_desc records; every offset/size must be a multiple of 16 bytes.
 * ---------------------------------------------------------------------- */
typedef struct ssb_copy_desc {
  int64_t src_off;    /* bytes from src base                          */
  int64_t dst_off;    /* bytes from dst base                          */
  int64_t src_stride; /* bytes between rows                           */
  int64_t dst_stride; /* bytes between rows                           */
  int64_t cum_bytes;  /* exclusive prefix of rows*row_bytes over descs */
  int32_t rows;
  int32_t row_bytes;
} ssb_copy_desc;

/* total_bytes = sum of rows*row_bytes = cum_bytes[n-1] + last size.
 * dst == NULL: every dst_off is an absolute device address (e.g. a peer's
 * receive buffer mapped over NVLink), the weight re-partition's P2P path. */
int ssb_copy2d_batched(const void* src, void* dst, const ssb_copy_desc* descs, int n_desc,
                       int64_t total_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Host KV tier staging (swap-out gather K3 / swap-in scatter K4).
 * Replaces the swap transfer charges of the reference: swap-out
 * sum(kv)/out_bw overlapped with prefill (sim.py:382-385) and the prefetcher's
 * swap-in at in_bw (sim.py:436-504), in the HND host layout
 * (reshard.py:191-201).
 * One sequence's KV in this GPU's pool (blocks[0:n_blocks], n_tokens tokens)
 * <-> contiguous HND staging [nl][2][nh][n_tokens][head_dim] covering pool
 * layers [l0, l0+nl) and heads [h0, h0+nh).  gather=1: pool -> staging,
 * gather=0: staging -> pool.  The caller moves staging <-> pinned host memory
 * with cudaMemcpyAsync on its copy stream. */
int ssb_kv_hnd_copy(int gather, void* pool, ssb_kv_geometry geo, const int32_t* blocks,
                    int n_blocks, int n_tokens, int l0, int nl, int h0, int nh, void* staging,
                    void* stream);

/* Strided host<->device copy (cudaMemcpy2DAsync, direction inferred from
 * the pointers; host memory must be pinned/registered for asynchrony):
 * `height` rows of `width` bytes.  Moves a GPU's (layer x head) rectangle
 * of a sequence between the staging buffer and the shared host-tier slot. */
int ssb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                       int64_t height, void* stream);

/* ------------------------------------------------------------------------
 * Deterministic weight initialisation (counter-based; see csrc/init.cu).
 * Not a reference op: it lets every GPU build its own shard of the
 * random-init model (synthetic weights) bit-identically to the
 * CPU oracle.  `segs` is a DEVICE array; element (r, c) of segment s is
 * arena[dst_off + r*ld + c] = value(seed, tensor_id, (row0+r)*full_cols + col0+c).
 * ---------------------------------------------------------------------- */
typedef struct ssb_init_seg {
  int64_t dst_off;   /* elements into the arena                 */
  int64_t ld;        /* destination row stride (elements)       */
  int64_t row0;      /* logical origin                          */
  int64_t col0;
  int64_t full_cols; /* logical tensor width                    */
  int64_t cum_elems; /* exclusive prefix of rows*cols           */
  int32_t rows;
  int32_t cols;
  int32_t tensor_id;
  float scale;       /* std; 0 => constant 1.0 (norm gains)    */
} ssb_init_seg;

int ssb_init_weights(void* arena, const ssb_init_seg* segs, int n_seg, int64_t total_elems,
                     uint64_t seed, void* stream);

/* ------------------------------------------------------------------------
 * Transformer-layer element ops (no reference counterpart: the reference
 * cost model does not price them).
 * ---------------------------------------------------------------------- */
/* out[r,:] = x[i,:] * rsqrt(mean(x[i]^2)+eps) * w with i = row_idx ? row_idx[r] : r
 * (bf16 in/out, fp32 math; row_idx gathers e.g. the last token of each
 * prompt before the LM head) */
int ssb_rmsnorm(const void* x, int ldx, const int32_t* row_idx, const void* w, void* out, int ldo,
                int rows, int hidden, float eps, void* stream);

/* ------------------------------------------------------------------------
 * TP combine over NVLink peer memory fused with the following RMSNorm
 * (replaces the NCCL all-reduce of the row-parallel o_proj / down_proj
 * partials that the reference charges per layer, perf.py:71-74 /
 * SURVEY.md §8(e), plus the rmsnorm launch after it).
 *
 * Every *_addrs argument is a HOST array of nranks device addresses valid in
 * the calling process (own buffer at [rank], CUDA IPC mappings of the peers'
 * buffers elsewhere; comm.peer_addresses):
 *   part[r]  bf16 [rows, ld]  rank r's partial sums (rank 0's include the residual)
 *   x[r]     bf16 [rows, ld]  receives x = sum_r part[r] (fp32 sum in rank order, bf16)
 *   h[r]     bf16 [rows, ld]  receives rmsnorm(x) * gamma   (h_addrs/gamma may be NULL)
 *   sig[r]   ssb_tp_signal_bytes() of zero-initialised device memory per rank
 * Rank r reduces rows [r*rows/n, (r+1)*rows/n) and stores them to every rank.
 * All ranks must make the same calls with the same (rows, hidden, ld,
 * max_blocks).  epoch 0 (what the engine passes): the epochs live in the
 * signal buffer, one counter per CTA index, advanced by the kernel itself —
 * so a call captured in a CUDA graph stays correct at every replay.  A
 * non-zero epoch (starting at 1, growing by one per call, never mixed with
 * epoch-0 calls on the same signal buffer) is taken from the host instead.
 * The call synchronises with the peers on the device (no host round trip).
 * A peer missing for 30 s sets *err = 1 (traps if err is NULL).
 * hidden <= 8192, nranks <= 8.
 * ---------------------------------------------------------------------- */
size_t ssb_tp_signal_bytes(void);
int ssb_tp_allreduce_rmsnorm(const uint64_t* part_addrs, const uint64_t* x_addrs, const uint64_t* h_addrs,
                             const uint64_t* sig_addrs, int nranks, int rank, int rows, int hidden, int ld,
                             const void* gamma, float eps, uint32_t epoch, int max_blocks, uint32_t* err,
                             void* stream);

/* The same combine for the folded-norm layout: x[:rows] <- sum of the
 * ranks' partials on every rank (as above), and instead of h the per-row
 * fp32 sum of squares of the stored bf16 x -- the reduction rmsnorm uses --
 * into every rank's ss[rows]; the consumer GEMMs apply 1/rms from it
 * (ssb_rownorm with ss_in_parts = 1) with the gains folded into their
 * weights.  Halves the bytes each rank stores over NVLink. */
int ssb_tp_allreduce_rowss(const uint64_t* part_addrs, const uint64_t* x_addrs, const uint64_t* ss_addrs,
                           const uint64_t* sig_addrs, int nranks, int rank, int rows, int hidden, int ld,
                           uint32_t epoch, int max_blocks, uint32_t* err, void* stream);

/* Vocab-parallel greedy token of every row across the TP group over peer
 * memory (replaces the (max, idx) all-gathers + ssb_argmax_combine the
 * reference's TP decode implies): keys[r] is rank r's uint64 [rows] from
 * ssb_gemm_lm_head_argmax (orderable logit << 32 | ~global index); out_idx
 * [rows] receives the index of the largest key over all ranks (the largest
 * logit, lowest index on ties).  Same signal buffer, epoch and error rules
 * as ssb_tp_allreduce_rmsnorm (the two share the per-CTA epoch counters). */
int ssb_tp_argmax_keys(const uint64_t* key_addrs, const uint64_t* sig_addrs, int nranks, int rank, int rows,
                       int32_t* out_idx, uint32_t epoch, int max_blocks, uint32_t* err, void* stream);

/* Decode-step bookkeeping on device: ctx_lens[b] += 1; positions[b] =
 * ctx_lens[b]-1; slots[b] = block_tables[b][pos/bs]*bs + pos%bs. */
int ssb_decode_positions(int32_t* ctx_lens, const int32_t* block_tables, int max_blocks,
                         int block_size, int32_t* positions, int64_t* slots, int batch,
                         void* stream);

/* In place RoPE (rotate-half) of the q and k heads of qkv[T, (nq+2nk)*d]
 * (row stride ld) at positions[t] using the fp32 tables cos/sin[max_pos][d/2],
 * then append k and v of every token to the paged pool at slot
 * slots[t] = block*block_size + offset, local layer `layer`.  A negative slot
 * skips the append (padding rows). */
int ssb_rope_kv_append(void* qkv, int ld, int T, int nq, int nk, const int32_t* positions,
                       const float* rope_cos, const float* rope_sin, int max_pos, void* pool,
                       ssb_kv_geometry geo, int layer, const int64_t* slots, void* stream);

/* Vocab-parallel embedding gather: out[t,:] = table[ids[t]-vocab_begin,:]
 * when the id falls in [vocab_begin, vocab_begin+vocab_local), else zeros. */
int ssb_embedding(const int32_t* ids, int T, const void* table, int vocab_begin, int vocab_local,
                  int hidden, void* out, int ldo, void* stream);

/* Per-row argmax of fp32 logits [rows, cols] (row stride ld); ties resolve to
 * the smallest index; out_idx = index_base + column. */
int ssb_argmax_rows(const float* logits, int ld, int rows, int cols, int index_base, float* out_val,
                    int32_t* out_idx, void* stream);

/* LM head fused with the greedy argmax: keys[m] = packed (max over the
 * N columns of A[m].B^T, smallest index of the max + index_base), never
 * materialising the fp32 logits (M x N x 4 bytes).  keys are zeroed by the
 * call (stream-ordered) and filled by 64-bit atomicMax from every tile.
 * Same values and tie rule as ssb_gemm_bf16(SSB_EPI_F32) + ssb_argmax_rows.
 * Workspace as for ssb_gemm_bf16_ws. */
int ssb_gemm_lm_head_argmax(const void* A, const void* B, int M, int N, int K, int lda, int ldb,
                            int index_base, unsigned long long* keys, int block_n, int max_ctas,
                            void* workspace, int64_t workspace_bytes, ssb_rownorm* rn, void* stream);
/* keys -> (value, index) arrays for ssb_argmax_combine / the token ids. */
int ssb_argmax_keys_decode(const unsigned long long* keys, int rows, float* out_val, int32_t* out_idx,
                           void* stream);

/* Combine n_parts partial argmaxes laid out [n_parts][rows] (vocab-parallel
 * lm_head): largest value, smallest index on ties. */
int ssb_argmax_combine(const float* vals, const int32_t* idxs, int n_parts, int rows,
                       int32_t* out_idx, void* stream);

/* ------------------------------------------------------------------------
 * Attention.  Replaces perf.py:68-89 / :92-111 (attention traffic and
 * compute) in _quantum (sim.py:335-341).
 * ---------------------------------------------------------------------- */
/* Causal prefill over packed sequences: qkv[total_tokens, (nq+2nk)*d] (RoPE
 * applied), sequence s spans rows [cu_seqlens[s], cu_seqlens[s+1]);
 * out[T, nq*d].  variant 0 = auto (persistent tcgen05/TMEM kernel for
 * head_dim 128), 1 = the mma.sync kernel (head_dim 64 always uses it),
 * 2 = the tcgen05 kernel with one CTA per (query tile, head, sequence). */
int ssb_prefill_attention(const void* qkv, int ld, int total_tokens, int nq, int nk, int head_dim,
                          const int32_t* cu_seqlens, int nseq, int max_len, void* out, int ldo,
                          float softmax_scale, int variant, void* stream);

/* Paged GQA decode, one query token per sequence: q = qkv[b, 0:nq*d];
 * K/V of local layer `layer` read from the pool through
 * block_tables[b][0:ceil(ctx_lens[b]/64)] (block_size must be 64);
 * out[b, nq*d]. */
int ssb_decode_attention(const void* qkv, int ld, int nq, int nk, const void* pool,
                         ssb_kv_geometry geo, int num_blocks, int layer, const int32_t* block_tables,
                         int max_blocks, const int32_t* ctx_lens, int batch, void* out, int ldo,
                         float softmax_scale, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SEESAW_B200_H_ */
