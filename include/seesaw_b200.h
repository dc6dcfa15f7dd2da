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

const char* ssb_last_error(void);
int ssb_version(void);
int ssb_device_sm_count(void);

/* ------------------------------------------------------------------------
 * Dense projections (bf16 tcgen05/TMEM GEMM fed by TMA).
 * Replaces perf.py:59-65 (linear weight traffic) and perf.py:92-111 (linear
 * compute) in _quantum (sim.py:335-341).
 * C[M,N] = A[M,K] . B[N,K]^T with A, B K-major.  block_n = 0 picks the tile.
 * ---------------------------------------------------------------------- */
int ssb_gemm_bf16(const void* A, const void* B, void* C, const void* R, int M, int N, int K,
                  int lda, int ldb, int ldc, int ldr, int epilogue, int block_n, void* stream);

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

int ssb_kv_reshard_pack(const void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                        int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                        const int32_t* nh, const int64_t* off_bytes, void* staging, void* stream);
int ssb_kv_reshard_unpack(void* pool, ssb_kv_geometry geo, const int32_t* block_ids, int n_ids,
                          int n_peers, const int32_t* l0, const int32_t* nl, const int32_t* h0,
                          const int32_t* nh, const int64_t* off_bytes, const void* staging,
                          void* stream);

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

/* total_bytes = sum of rows*row_bytes = cum_bytes[n-1] + last size. */
int ssb_copy2d_batched(const void* src, void* dst, const ssb_copy_desc* descs, int n_desc,
                       int64_t total_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SEESAW_B200_H_ */
