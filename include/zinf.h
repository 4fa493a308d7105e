/* libzinf — C ABI of the B200-native ZeRO-Infinity partitioned data-parallel step.
 *
 * Drop-in boundary for the reference `infinisim` hot path (/root/reference).
 * The reference is pure Python + numpy (pkg/pyproject.toml:10-12); the
 * Python mirror `paper_2104_07857_b200` keeps its API and calls these
 * entry points through ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - Every call returns a zi_status; on failure zi_last_error() holds a
 *     thread-local message. Status codes map to the reference exception tree
 *     (store.py:54-71): ZI_ECAPACITY -> CapacityExceeded, ZI_ENOTFOUND ->
 *     KeyNotFound, ZI_EINVAL -> ValueError, ZI_EEXHAUSTED -> PoolExhausted,
 *     ZI_EIO -> OSError, ZI_ECUDA/ZI_ENCCL -> StoreError.
 *   - All device work is asynchronous on the caller's `stream`
 *     (a cudaStream_t passed as void*). Callers own every buffer; the
 *     library owns nothing but its error string.
 *   - Element counts are size_t; pointers are device pointers unless noted.
 *   - half_kind: ZI_HALF_FP16 (SPEC parity type) or
 *     ZI_HALF_BF16 (BASELINE configs).
 */
#ifndef ZINF_H
#define ZINF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ZI_OK = 0,
  ZI_EINVAL = 1,
  ZI_ECAPACITY = 2,
  ZI_ENOTFOUND = 3,
  ZI_ECUDA = 4,
  ZI_ENCCL = 5,
  ZI_EEXHAUSTED = 6,
  ZI_EIO = 7
} zi_status;

enum { ZI_HALF_FP16 = 0, ZI_HALF_BF16 = 1 };

/* Element types, numbered as the reference shard format's dtype byte
 * (store.py:37: 0 = f32, 1 = f16, 2 = f64) plus this build's 3 = bf16. */
enum { ZI_DT_F32 = 0, ZI_DT_F16 = 1, ZI_DT_F64 = 2, ZI_DT_BF16 = 3 };

/* Adam constants folded on the host in float32 exactly as oracle/adam.py
 * AdamConsts.make does: lr, beta1, 1-beta1, beta2, 1-beta2, 1-beta1^t,
 * 1-beta2^t, eps. */
typedef struct {
  float lr, b1, omb1, b2, omb2, bc1, bc2, eps;
} zi_adam_consts;

const char* zi_last_error(void);
int zi_version(void);

/* ---- optimizer ------------------------------------------------------------
 * chunked_adam_step for one chunk: in place on fp32
 * p/m/v with fp32 gradient g, writes the RNE half copy of p to p_half
 * (may be NULL). Bit-exact with oracle/adam.py:adam_update. */
int zi_adam_step(float* p, float* m, float* v, const float* g, void* p_half,
                 size_t n, const zi_adam_consts* c, int half_kind, void* stream);

/* ---- collectives ----------------------------------------------------------
 * reduce_scatter fused with the half->fp32 cast and scale (SPEC.md:484-492,
 * SPEC.md:750,782). contribs[k] (k = 0..n_contrib-1, in fold order) are
 * full-length half gradient buckets, local or IPC-mapped peer memory.
 *   out[i] = scale * fold_k fp32(contribs[k][shard_offset + i]),
 * the fold being a left-to-right fp32 sum; elements at or beyond
 * contrib_len read as 0 (zero pad of the last shard). */
int zi_reduce_scatter_cast(const void* const* contribs, int n_contrib,
                           size_t shard_offset, size_t shard_elems, size_t contrib_len,
                           float scale, int half_kind, float* out, void* stream);

/* reduce_scatter for any SPEC dtype: half inputs as
 * zi_reduce_scatter_cast (fp32 out); f32 folds in fp32, f64 in fp64 (out
 * has the input type). scale multiplies the folded sum. */
int zi_reduce_scatter(const void* const* contribs, int n_contrib, size_t shard_offset,
                      size_t shard_elems, size_t contrib_len, int dtype, double scale,
                      void* out, void* stream);

/* The engine's per-layer update: zi_reduce_scatter_cast followed by
 * zi_adam_step in one pass over HBM (no fp32 gradient round trip).
 * g_out (nullable) receives the fp32 gradient shard for parity tests. */
int zi_rs_adam(const void* const* contribs, int n_contrib, size_t shard_offset,
               size_t shard_elems, size_t contrib_len, float scale, int half_kind,
               float* p, float* m, float* v, void* p_half, float* g_out,
               const zi_adam_consts* c, void* stream);

/* zi_rs_adam with the Adam constants read from device memory (c_dev), so a
 * captured CUDA graph replays with per-step bias corrections. */
int zi_rs_adam_dc(const void* const* contribs, int n_contrib, size_t shard_offset,
                  size_t shard_elems, size_t contrib_len, float scale, int half_kind,
                  float* p, float* m, float* v, void* p_half, float* g_out,
                  const zi_adam_consts* c_dev, void* stream);

/* Device-side step advance: *step_dev += 1, then *consts_dev = the constants
 * of that step folded exactly as on the host (double math, one rounding). */
int zi_adam_advance(double lr, double beta1, double beta2, double eps, int* step_dev,
                    zi_adam_consts* consts_dev, void* stream);

/* allgather: full[r*shard_elems + i] = shards[r][i],
 * truncated to full_elems. shards[r] may be IPC-mapped peer memory.
 * elem_bytes in {2,4,8}. use_copy_engine != 0 issues one cudaMemcpyAsync per
 * rank (zero SMs); otherwise one vectorised SM copy kernel. */
int zi_allgather(const void* const* shards, int world, size_t shard_elems,
                 size_t elem_bytes, void* full, size_t full_elems,
                 int use_copy_engine, void* stream);

/* Cross-GPU barrier over IPC-mapped flag words: rank writes `epoch` into
 * slot [rank] of every peer's flag array (flags[k] = peer k's array of
 * `world` uint32), then spins until its own array holds >= epoch in every
 * slot. Orders the P2P reduce-scatter / gather with the peers' producers. */
int zi_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch, void* stream);
/* Same barrier with the epoch taken from (and advanced in) a device counter: graph-safe. */
int zi_barrier_dev(uint32_t* const* flags, int world, int rank, uint32_t* epoch_ctr,
                   void* stream);

/* ---- init / casts ---------------------------------------------------------
 * Counter-RNG uniform init (oracle/numerics.py:uniform_init):
 * master[i] = float32(2k+1-2^24) * scale with k = top 24 bits of
 * splitmix64(key + (start_index+i+1)*golden); p_half[i] = RNE(master[i]).
 * Either output may be NULL. */
int zi_init_uniform(float* master, void* p_half, size_t n, uint64_t key,
                    uint64_t start_index, float scale, int half_kind, void* stream);
int zi_fill(float* master, void* p_half, size_t n, float value, int half_kind,
            void* stream);
int zi_cast_f32_to_half(const float* src, void* dst, size_t n, int half_kind,
                        void* stream);
int zi_cast_half_to_f32(const void* src, float* dst, size_t n, int half_kind,
                        void* stream);

/* C[m,n] = sum_{k=0..K-1} A[m,k] B[k,n] (+ bias[n]) in fp32 or fp64 (dtype ZI_DT_F32 /
 * ZI_DT_F64), one sequential fma chain per output: a fixed summation order, independent
 * of library heuristics. Strides in elements (A: sam, sak; B: sbk, sbn; C: scm, scn), so
 * transposed views cost nothing. bias may be NULL. The SPEC harness's linears
 * ("fixed order everywhere") run on it so that AC-9's
 * digests are bit-identical across world sizes and placements. */
int zi_matmul_fixed(const void* A, int64_t sam, int64_t sak, const void* B, int64_t sbk,
                    int64_t sbn, const void* bias, void* C, int64_t scm, int64_t scn, int M,
                    int N, int K, int dtype, void* stream);

/* ---- fused block kernels of the GPT step (bf16 activations, fp32 math) ----
 * Row-wise ops take T rows of H (H in {128, 256, 512, 1024, 2048}); column
 * reductions are deterministic (fixed-order fold of per-CTA partials in the
 * caller's fp32 `work` buffer). Gradient outputs are bf16 (RNE of the fp32
 * sum) or fp32 when *_f32 != 0.
 *   zi_ln_fwd     y = (x [+ resid] - mean) * rstd * w + b; with resid, also
 *                 xsum = bf16(x + resid) (residual add fused); mean/rstd per row.
 *   zi_ln_bwd     dx = rstd * (dy*w - mean(dy*w) - xh * mean(dy*w*xh)) [+ dres];
 *                 dgamma = sum_rows dy * xh, dbeta = sum_rows dy; with dres_sum,
 *                 also dres_sum = sum_rows dres (the bias gradient of the linear
 *                 whose output gradient is dres), all from one pass.
 *   zi_gelu_fwd   y = gelu_tanh(u) over n bf16 (n % 8 == 0; SFU tanh, the error is
 *                 below bf16 output precision).
 *   zi_bias_grad  db = sum_rows dy; with u given, first du = gelu_tanh'(u) * dy
 *                 (stored to du) and db = sum_rows du.
 *   zi_softmax_ce in place over T rows of V bf16 logits: loss_rows = lse - l[t],
 *                 logits <- (softmax - onehot(t)) * scale; *loss = mean(loss_rows). */
int zi_ln_fwd(const void* x, const void* resid, void* xsum, const void* w, const void* b, void* y,
              float* mean, float* rstd, int T, int H, float eps, void* stream);
int zi_ln_bwd(const void* dy, const void* x, const void* w, const float* mean, const float* rstd,
              const void* dres, void* dx, void* dgamma, void* dbeta, void* dres_sum, int grads_f32,
              float* work, size_t work_elems, int T, int H, void* stream);
int zi_gelu_fwd(const void* u, void* y, size_t n, void* stream);
int zi_bias_grad(const void* dy, const void* u, void* du, void* db, int db_f32, float* work,
                 size_t work_elems, int T, int N, void* stream);
int zi_softmax_ce(void* logits, const int64_t* targets, float* loss_rows, float* loss, int T,
                  int V, float scale, void* stream);

/* Kernels libzinf has launched in this process (every entry point counts its launches,
 * including launches recorded into a CUDA graph during capture). Diagnostics. */
long long zi_launch_count(void);

/* ---- offload engine (tier-store host tier, store.py:81-153) -------------- */
int zi_host_alloc(size_t bytes, void** out);          /* pinned, portable */
int zi_host_free(void* p);
/* kind: 0 H2D, 1 D2H, 2 D2D, 3 default (UVA) */
int zi_memcpy_async(void* dst, const void* src, size_t bytes, int kind, void* stream);
int zi_event_create(void** ev);                       /* timing disabled */
int zi_event_destroy(void* ev);
/* Timing events that survive CUDA-graph capture: an external record node is
 * re-recorded on every replay, so kernel durations inside a graphed step are
 * measured with CUDA events on the launching stream. */
int zi_event_create_timed(void** ev);
int zi_event_record_external(void* ev, void* stream);
int zi_event_elapsed_ms(void* ev0, void* ev1, float* ms);
int zi_event_record(void* ev, void* stream);
int zi_event_query(void* ev);                         /* ZI_OK done, ZI_ENOTFOUND pending */
int zi_event_sync(void* ev);
int zi_stream_wait_event(void* stream, void* ev);

/* Staging-buffer pool: the reference BufferPool (store.py:81-123). buffer_count
 * buffers of buffer_bytes, pinned (cudaHostAlloc) or pageable (pinned = 0, hosts
 * without a GPU). acquire hands out buffer indices LIFO; when none is free it
 * blocks (blocking = 1; counted in waits) or returns ZI_EEXHAUSTED. release
 * returns ZI_EINVAL for an index outside the pool ("does not belong") or when
 * every buffer is already free ("over-released"). Thread-safe. */
int zi_pool_create(size_t buffer_bytes, int buffer_count, int blocking, int pinned, void** pool);
int zi_pool_destroy(void* pool);
int zi_pool_buffer(void* pool, int index, void** ptr);
int zi_pool_acquire(void* pool, int* index);
int zi_pool_release(void* pool, int index);
int zi_pool_stats(void* pool, int* free_count, uint64_t* waits);

/* The offload lanes: one async copy on `stream`, then `event`
 * (nullable, a zi_event_create event) recorded behind it — the IoTicket of
 * store.py:126-153. H2D = cg-transfer (host tier -> HBM prefetch slot),
 * D2H = grad / optimizer-state offload. Pinned host memory for full speed. */
int zi_h2d_async(void* dst, const void* src, size_t bytes, void* stream, void* event);
int zi_d2h_async(void* dst, const void* src, size_t bytes, void* stream, void* event);

/* ---- native file I/O for the NVMe tier (store.py:442-560, PAPER §6.2) ---------
 * A worker pool moving byte ranges of a file between disk and pinned host memory.
 * zi_aio_open opens the file twice: fds[0] O_DIRECT, fds[1] buffered. zi_aio_submit
 * queues file bytes [b0, b1) <-> buf + (b0 % 4096) ... (buf 4 KiB-aligned): whole 4 KiB
 * blocks go O_DIRECT in <= 8 MiB pieces across the workers, partial edge blocks through
 * the buffered descriptor; zi_aio_wait blocks until that request finished (ZI_EIO on an
 * I/O error or a short read). */
int zi_aio_create(int threads, void** eng);
int zi_aio_destroy(void* eng);
int zi_aio_open(const char* path, int write, int create, int* fds);
int zi_aio_close(const int* fds);
int zi_aio_truncate(const int* fds, size_t size);
int zi_aio_submit(void* eng, const int* fds, int write, void* buf, size_t b0, size_t b1,
                  uint64_t* id);
int zi_aio_wait(void* eng, uint64_t id);

/* ---- CUDA IPC (peer buffers for the P2P collectives) ---------------------
 * Buffers that peers map are plain cudaMalloc allocations (zi_device_alloc)
 * so the IPC handle names exactly that buffer (offset 0). */
int zi_device_alloc(size_t bytes, void** out);
int zi_device_free(void* p);
int zi_ipc_get_handle(void* dptr, unsigned char handle[64]);
int zi_ipc_open(const unsigned char handle[64], void** dptr);
int zi_ipc_close(void* dptr);

/* ---- communicator context (SURVEY.md §8(b) zi_ctx_create / zi_ctx_destroy) -
 * One per data-parallel rank: rank, world, device, and "windows" = the same-shaped
 * buffer on every rank (parameter arena, gradient ring, barrier flags), IPC-mapped
 * into this process once. Handles and byte offsets are exchanged out of band
 * (torch.distributed in comm.DistComm): handles = world x 64 bytes from
 * zi_ipc_get_handle of each rank's allocation, offsets = world byte offsets of the
 * window inside it (our own entries are ignored; `local` is our pointer). The
 * collectives below are the SPEC ops over a window, rank order = fold order.
 * The NCCL communicator is torch.distributed's (plumbing); the data path is
 * P2P loads/stores and copy-engine DMA over NVLink. Replaces the reference's
 * in-process rank loop. Thread-safe per context. */
typedef struct zi_ctx zi_ctx;
int zi_ctx_create(int rank, int world, int device, zi_ctx** out);
int zi_ctx_destroy(zi_ctx* ctx);
int zi_ctx_info(const zi_ctx* ctx, int* rank, int* world, int* device);
int zi_ctx_add_window(zi_ctx* ctx, void* local, const unsigned char* handles,
                      const uint64_t* offsets, int* win);
int zi_ctx_window_ptrs(zi_ctx* ctx, int win, void** ptrs);
/* SPEC allgather: full[r*shard + i] = window_r[offset + i]. */
int zi_ctx_allgather(zi_ctx* ctx, int win, size_t offset_bytes, size_t shard_elems, int dtype,
                     void* full, size_t full_elems, int use_copy_engine, void* stream);
/* SPEC reduce_scatter + cast: our shard (rank * shard_elems ..)
 * of the rank-order fp32 fold of every rank's half bucket at window + offset,
 * times scale; elements >= contrib_len read 0. Bit-exact to the oracle. */
int zi_ctx_reduce_scatter_cast(zi_ctx* ctx, int win, size_t offset_bytes, size_t contrib_len,
                               size_t shard_elems, float scale, int half_kind, float* shard_out,
                               void* stream);
/* zi_barrier_dev over a window of `world` uint32 flags; the epoch is a device counter per
 * window, so the barrier may be captured in a CUDA graph and replayed. */
int zi_ctx_barrier(zi_ctx* ctx, int flags_win, void* stream);
/* Barrier with no SM held, over a flag window of 2*world uint32 (two slot sets). Arrive =
 * cuStreamWriteValue32(1) into our slot of set `parity` in every peer's array (fenced
 * after this stream's earlier writes); wait = cuStreamWaitValue32(== 1) on every peer's
 * slot of our set in the stream front end, then reset it to 0. Consecutive barriers on
 * one window alternate parity; comm.DistComm keeps that order, padding a captured CUDA
 * graph to an even barrier count per window. */
int zi_ctx_barrier_value(zi_ctx* ctx, int flags_win, int parity, void* stream);

/* ---- memory-centric tiling ------------------------------
 * One tile of a tiled linear on the 5th-gen tensor cores (tcgen05 + TMEM,
 * TMA-fed), bf16 in, fp32 accumulate, bf16 out:
 *   y[m, n] = sum_k x[m, k] * w[n, k] + bias[n]     (bias nullable)
 * x: M x K row-major (ld = ldx elements), w: N x K row-major (ldw), y: M x N
 * (ldy). Requires K % 64 == 0, ldx/ldw/ldy % 8 == 0, 16-byte aligned bases. */
int zi_linear_fwd(const void* x, const void* w, const void* bias, void* y,
                  int M, int N, int K, int ldx, int ldw, int ldy, void* stream);

/* One tile of TiledLinear, the §8(b) names. Tile t holds rows
 * [s, e) of W, so N_t = e - s:
 *   fwd: y_t[m, n] = sum_k x[m, k] w_t[n, k] + b_t[n]       (zi_linear_fwd)
 *   bwd: dw_t[n, k] = sum_m dy_t[m, n] x[m, k]               (bf16, ld lddw; NULL skips)
 *        dx_acc[m, k] += sum_n dy_t[m, n] w_t[n, k]          (fp32, ld lddx; NULL skips)
 *        db_t[n] = sum_m dy_t[m, n]                          (fp32, fixed order; NULL skips)
 * dy_t is the tile's column block of the upstream gradient (ld lddy), so tiles
 * are processed in order with dx accumulated sequentially. */
int zi_linear_tile_fwd(const void* x, const void* w_t, const void* b_t, void* y, int M, int K,
                       int N_t, int ldx, int ldw, int ldy, void* stream);
int zi_linear_tile_bwd(const void* x, int ldx, const void* w_t, int ldw, const void* dy_t,
                       int lddy, void* dw_t, int lddw, float* dx_acc, int lddx, float* db_t,
                       int M, int K, int N_t, void* stream);

/* General tcgen05 GEMM behind the tiled linear's forward and backward:
 *   D[m, n] = sum_k A(m, k) * B(n, k) (+ bias[n]) (+ D[m, n] if accumulate)
 * A(m, k) = A[m*lda + k] (a_mn_major = 0) or A[k*lda + m] (a_mn_major = 1);
 * B(n, k) = B[n*ldb + k] or B[k*ldb + n]. bf16 operands, fp32 accumulate;
 * D is bf16 (d_f32 = 0) or fp32 (d_f32 = 1), row-major with ldd.
 * Supported (a_mn, b_mn, d_f32, accumulate): (0,0,0,0) forward,
 * (0,1,0,0) / (0,1,1,0) / (0,1,1,1) input gradient dx = dy W,
 * (1,1,0,0) / (1,1,1,0) weight gradient dW = dy^T x, (0,0,1,0/1). */
int zi_gemm(const void* A, int a_mn_major, int lda, const void* B, int b_mn_major, int ldb,
            const void* bias, void* D, int d_f32, int accumulate, int ldd,
            int M, int N, int K, void* stream);

/* The same GEMM with a fused bf16 epilogue (the GPT block's linears; no
 * reference counterpart, a build extension of the SPEC's tile GEMM):
 *   ZI_EPI_PLAIN  D = acc (+ bias)
 *   ZI_EPI_GELU   D = u = bf16(acc + bias), D2 = bf16(gelu_tanh(u))   fc1 forward
 *   ZI_EPI_RESID  D = bf16(bf16(acc + bias) + X)                        fc2 forward + residual
 *   ZI_EPI_DGELU  D = bf16(bf16(acc) * gelu_tanh'(X)), X = u            fc2 dX -> fc1 du
 * zi_gemm_sk only:
 *   ZI_EPI_GELU_SAVE  u = bf16(acc + bias): D = bf16(gelu_tanh'(u)), D2 = bf16(gelu_tanh(u))
 *                     (fc1 forward keeping GELU' for the backward instead of u)
 *   ZI_EPI_MUL        D = bf16(bf16(acc) * X), X = the saved GELU'           fc2 dX -> fc1 du
 * X (ldx) and D2 (ldd2) are M x N bf16; N % 8 == 0 and all leading dimensions
 * multiples of 8. Operand majorness as zi_gemm. */
enum { ZI_EPI_PLAIN = 0, ZI_EPI_GELU = 1, ZI_EPI_RESID = 2, ZI_EPI_DGELU = 3,
       ZI_EPI_GELU_SAVE = 4, ZI_EPI_MUL = 5 };
int zi_gemm_ex(const void* A, int a_mn_major, int lda, const void* B, int b_mn_major, int ldb,
               const void* bias, void* D, int ldd, const void* X, int ldx, void* D2, int ldd2,
               int epi, int M, int N, int K, void* stream);
/* Stream-K GEMM behind the GPT step's linears (csrc/gemm_sk.cu): 2-SM 256 x 256 pair
 * tiles, two TMEM accumulators, and a hybrid stream-K schedule that deals the last
 * waves' k-blocks evenly over the CTA pairs. Same operands and epilogues as
 * zi_gemm_ex; d_f32 = 1 writes fp32 D (epi = ZI_EPI_PLAIN, no bias). ws (256-byte
 * aligned, >= zi_gemm_sk_workspace_bytes(), zeroed once before first use; its flags
 * reset themselves) enables the split; ws = NULL runs whole tiles. One workspace per
 * stream: launches sharing one must be stream-ordered. Results are deterministic
 * (partials summed in a fixed order) for a given device. */
size_t zi_gemm_sk_workspace_bytes(void);
int zi_gemm_sk(const void* A, int a_mn_major, int lda, const void* B, int b_mn_major, int ldb,
               const void* bias, void* D, int ldd, int d_f32, const void* X, int ldx, void* D2,
               int ldd2, int epi, int M, int N, int K, void* ws, size_t ws_bytes, void* stream);
/* zi_gemm_sk with epilogue side outputs of the bf16 result (NULL = off):
 *   colsum_part fp32 [ceil(M/32)][N]: column sums of each 32-row block of the stored bf16
 *     output (zi_colsum_fold then sums the blocks in order: a bias gradient, e.g. the fc1
 *     bias from the fc2 input-gradient GEMM with the GELU' epilogue);
 *   delta fp32 [B][H][S] (epi PLAIN, X = the attention output O, N = H * D, D 64 / 128,
 *     M = B * S): per row and head, the sum over the head's columns of bf16(D) * O, the
 *     attention backward's rowsum(dO o O) from the GEMM that produces dO. */
int zi_gemm_sk_aux(const void* A, int a_mn_major, int lda, const void* B, int b_mn_major, int ldb,
                   const void* bias, void* D, int ldd, int d_f32, const void* X, int ldx, void* D2,
                   int ldd2, int epi, int M, int N, int K, void* ws, size_t ws_bytes,
                   float* colsum_part, float* delta, int delta_S, int delta_H, int delta_D,
                   void* stream);
/* out[c] = sum over p < P of part[p][c] in p order (fp32 in; bf16 RNE or fp32 out). */
int zi_colsum_fold(const float* part, int P, int N, void* out, int out_f32, void* stream);
/* Deferred column folds (csrc/fused.cu). zi_ln_bwd_partials is zi_ln_bwd's row pass
 * alone: dx, and the per-CTA partials of dgamma, dbeta (and, with dres_sum != 0, of the
 * column sums of dres) as part fp32 [sets][P][H], P returned in *nparts (sets = 2 or 3).
 * zi_fold_sets then sums up to ZI_FOLD_MAX_SETS partial sets in one launch, each
 * out[c] = sum_p part[p * N + c] in the order zi_ln_bwd / zi_colsum_fold use (bitwise the
 * same results), so a block's four bias / LayerNorm gradient folds cost one launch. */
#define ZI_FOLD_MAX_SETS 8
typedef struct zi_fold_set {
  const float* part;   /* fp32 [P][N] */
  int P;
  int N;
  void* out;           /* [N], bf16 or fp32 (out_f32) */
} zi_fold_set;
int zi_ln_bwd_partials(const void* dy, const void* x, const void* w, const float* mean,
                       const float* rstd, const void* dres, void* dx, int dres_sum, float* part,
                       size_t part_elems, int T, int H, int* nparts, void* stream);
int zi_fold_sets(const zi_fold_set* sets, int n, int out_f32, void* stream);
/* Diagnostics: a device buffer of >= 148*16*8 u64 receiving clock64() stamps of the
 * wide-tile GEMM's pipeline (NULL turns it off). Not for production use. */
int zi_gemm_set_profile(void* buf);

/* ---- causal multi-head attention on tcgen05 (csrc/attn_sm100.cu) -------------
 * qkv [B*S, 3*H*D] bf16 (head h of q / k / v at columns h*D, H*D + h*D, 2*H*D + h*D),
 * out / dout [B*S, H*D] bf16, lse / delta fp32 [B*H*S] (lse in the log2 domain of the
 * scaled scores), dqkv like qkv. D in {64, 128}, S a multiple of 128. The backward
 * is deterministic: no atomics, every output row summed in a fixed order. */
int zi_attn_fwd(const void* qkv, void* out, float* lse, int B, int H, int S, int head_dim,
                void* stream);
int zi_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* delta,
                void* dqkv, int B, int H, int S, int head_dim, void* stream);
/* (out = NULL: delta already holds rowsum(dout o out), e.g. from zi_gemm_sk_aux.)
 * zi_attn_bwd_colsum also writes the column sums of dqkv (as stored, bf16) per 32-row
 * block into colsum_part, fp32 [B*S/32][3*H*D] — the qkv bias gradient's partials
 * (zi_colsum_fold sums them in block order). */
int zi_attn_bwd_colsum(const void* qkv, const void* out, const void* dout, const float* lse,
                       float* delta, void* dqkv, int B, int H, int S, int head_dim,
                       float* colsum_part, void* stream);
/* Tied-embedding gradient in a fixed order (csrc/embed.cu): out[v] = half_RNE(acc[v] +
 * sum of dx[t] over the tokens t with id v, in sequence order). tokens int64 [T]; dx
 * [T, hd] bf16 (dx_f32 = 0) or fp32; acc fp32 [V, hd]; out half [V, hd]; work int32
 * [2*V + 1 + T]. Deterministic: counting sort with stable ranks, no float atomics. */
int zi_embed_grad(const int64_t* tokens, int T, const void* dx, int dx_f32, const float* acc, int V,
                  int hd, void* out, int half_kind, int* work, void* stream);
/* Embedding lookup of the GPT forward (csrc/embed.cu), replacing torch's
 * F.embedding(tokens, wte) + wpe (the train_step forward): x[t] =
 * bf16_RNE(wte[tokens[t]] + wpe[t % S]) summed in fp32. tokens int64 [T]; wte bf16 [V, hd];
 * wpe bf16 [S, hd]; x bf16 [T, hd]. Ids outside [0, V) contribute no wte row. */
int zi_embed_fwd(const int64_t* tokens, int T, int S, const void* wte, const void* wpe, int V,
                 int hd, void* x, void* stream);
/* Position-embedding gradient in a fixed order: out[s] = sum over b = 0..B-1 (ascending)
 * of dx[b*S + s] in fp32; dx [B*S, hd] fp32 (dx_kind = -1) or half (ZI_HALF_*); out [S, hd] fp32
 * (out_kind = -1) or half RNE (ZI_HALF_BF16 / ZI_HALF_FP16) — the wpe gradient
 * contribution before the reduce-scatter. */
int zi_pos_grad(const void* dx, int dx_kind, int B, int S, int hd, void* out, int out_kind,
                void* stream);
/* Diagnostics: per-CTA globaltimer records of zi_attn_fwd into buf (6 u64 per CTA: sm,
 * entry, operands in, last MMA issued, softmax done, exit); NULL turns it off. */
int zi_attn_set_trace(void* buf);

#ifdef __cplusplus
}
#endif
#endif /* ZINF_H */
