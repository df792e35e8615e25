/* spl_c.h — C-ABI of the B200-native Spotlight decode-time retrieval path.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no
 * torch or C++ types. Every entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj). The reference's C++ API
 * (spotlight/bitcodes.hpp, hashers.hpp, attention_eval.hpp) is re-exposed on
 * top of this ABI by the C++ drop-in library (the headers under
 * include/spotlight/, libspotlight_b200.so), which marshals host<->device and re-throws the
 * reference exception types.
 *
 * Conventions
 *  - Unless a parameter says "host", every array pointer is DEVICE memory
 *    (cudaMalloc / torch CUDA tensors); `stream` is a cudaStream_t (NULL =
 *    legacy default stream). All kernels are asynchronous on `stream`.
 *  - A "problem" is one independent (batch, head) retrieval. Problem p reads
 *    its code rows at codes + p * problem_stride_rows * W (stride 0 = every
 *    problem shares one cache, as hash_topk's queries do) and its valid row
 *    count at n_valid[p / nvalid_div].
 *  - Code rows use the reference layout (bitcodes.hpp:50-92): W = L/32 u32
 *    words per row, column j in word j % W at bit 31 - j / W.
 *  - Status codes mirror the reference exceptions (errors.hpp:9-35);
 *    spl_last_error(ctx) returns the message of the last failure, worded as
 *    the reference words it (e.g. "top_k_indices: k=0 out of range for n=3").
 *  - A context owns a workspace and is NOT thread-safe: use one per host
 *    thread / stream (the reference functions are pure and concurrent-safe,
 *    SPEC.md:88-89; a context per caller keeps that property).
 */
#ifndef SPL_C_H
#define SPL_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum spl_status {
    SPL_OK = 0,
    SPL_E_DIMENSION = 1, /* DimensionError (errors.hpp:9-13) */
    SPL_E_NUMERIC = 2,   /* NumericError   (errors.hpp:21-25) */
    SPL_E_FORMAT = 3,    /* FormatError    (errors.hpp:15-19) */
    SPL_E_IO = 4,        /* IoError        (errors.hpp:32-35) */
    SPL_E_CUDA = 5,      /* CUDA runtime failure / no device */
    SPL_E_NCCL = 6,      /* collective failure (reported by host glue) */
    SPL_E_STATE = 7,     /* misuse: null handle, workspace during capture */
    SPL_E_EMPTY_PAIRS = 8 /* EmptyPairError (errors.hpp:27-30): no valid ranking pairs */
} spl_status;

typedef enum spl_dtype { SPL_F32 = 0, SPL_BF16 = 1, SPL_F64 = 2 /* spl_matmul / spl_map only */ } spl_dtype;
typedef enum spl_hasher_kind {
    SPL_HASHER_MLP = 1,
    SPL_HASHER_LINEAR = 0,
    SPL_HASHER_DOWNPROJ = 2 /* DownProjEstimator (training / evaluation only) */
} spl_hasher_kind;
typedef enum spl_encode_mode {
    SPL_ENCODE_EXACT = 0, /* CUDA cores, the reference's fmaf order + glibc expf: bit-exact */
    SPL_ENCODE_TC = 1     /* tcgen05 bf16 tensor cores, fp32 TMEM accumulation (bulk/prefill) */
} spl_encode_mode;

typedef struct spl_ctx spl_ctx;
typedef struct spl_hasher spl_hasher;

/* ---------------------------------------------------------------- context */
const char* spl_version(void);
spl_status spl_ctx_create(int device, spl_ctx** out);
void spl_ctx_destroy(spl_ctx* ctx);
const char* spl_last_error(const spl_ctx* ctx);
/* Pre-size the workspace for problems of up to (P, n_max, L, k) so that later
 * calls never allocate (required before CUDA-graph capture). */
spl_status spl_reserve(spl_ctx* ctx, uint32_t P, uint64_t n_max, uint32_t L, uint32_t k,
                       uint32_t d);
/* Device error word (non-finite encoder input -> NumericError, out-of-range
 * n_valid or append slot -> DimensionError, a retrieval whose CTAs could not
 * all run at once -> SPL_E_CUDA after the in-kernel 2 s watchdog: its indices
 * are then invalid). Kernels never fail the launch itself, so a caller that
 * replays captured decode steps should check this word at least once per
 * batch of steps. Synchronises `stream`, returns the recorded status and
 * clears it. */
spl_status spl_check_device_error(spl_ctx* ctx, void* stream);
/* Number of kernels this context launched so far (bench gpu_launches). */
uint64_t spl_launch_count(const spl_ctx* ctx);
/* Names of the kernels this context launched since the previous call, ';'-
 * separated (e.g. "k1_encode_cluster;k3_fused_pf;k4_gather;"), copied into buf
 * (host, NUL-terminated, truncated to len) and cleared. Returns the full
 * length. Lets tests assert which kernel variant a call ran. */
size_t spl_launch_log(spl_ctx* ctx, char* buf, size_t len);

/* memory helpers for callers that do not link the CUDA runtime (the C++
 * drop-in uses these; `kind`: 0 = default/UVA). */
spl_status spl_device_alloc(spl_ctx* ctx, size_t bytes, void** out);
spl_status spl_device_free(spl_ctx* ctx, void* p);
spl_status spl_memcpy(spl_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream);
spl_status spl_memset(spl_ctx* ctx, void* dst, int value, size_t bytes, void* stream);
spl_status spl_stream_synchronize(spl_ctx* ctx, void* stream);

/* --------------------------------------------------------------- bitcodes */
/* pack_bits (bitcodes.hpp:93, bitcodes.cpp:22-41): bits u8[n][L] -> codes
 * u32[n][L/32]. L % 32 != 0 or L == 0 -> SPL_E_DIMENSION. */
spl_status spl_pack_bits(spl_ctx* ctx, const uint8_t* bits, uint64_t n, uint32_t L,
                         uint32_t* codes, void* stream);
/* unpack_bits (bitcodes.hpp:96, bitcodes.cpp:43-57). */
spl_status spl_unpack_bits(spl_ctx* ctx, const uint32_t* codes, uint64_t n, uint32_t L,
                           uint8_t* bits, void* stream);
/* nxor_scores_into (bitcodes.hpp:103-104, bitcodes.cpp:59-76), batched:
 * scores[p][i] = sum_w popcount(~(q[p][w] ^ codes_p[i][w])) for i < n_valid
 * of problem p; scores row stride = scores_stride. Rows >= n_valid untouched. */
spl_status spl_nxor_scores(spl_ctx* ctx, const uint32_t* codes, uint64_t problem_stride_rows,
                           uint32_t L, const uint32_t* qcodes, uint32_t P,
                           const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                           int32_t* scores, uint64_t scores_stride, void* stream);
/* top_k_indices<S> (bitcodes.hpp:106-121, bitcodes.cpp:89-131) over P score
 * rows of n (device) each: the k best by (score desc, index asc), written
 * ascending to idx[p][0..k). k == 0 or k > n -> SPL_E_DIMENSION with the
 * reference's message. dtype: 0 = int32, 1 = float32, 2 = float64. */
spl_status spl_top_k(spl_ctx* ctx, const void* scores, int dtype, uint32_t P, uint64_t n,
                     uint64_t scores_stride, uint32_t k, uint32_t* idx, void* stream);

/* ------------------------------------------- dense retrieval */
/* oracle_topk (attention_eval.hpp:47, attention_eval.cpp:121-135): for every
 * problem p (one query q[p][d] against rows [0, n_valid) of keys + p * cap * d,
 * an f32/bf16 [.][cap][d] cache; cap = 0: every problem reads the same
 * rows, as the queries of one AttentionInstance do), the exact float
 * logits of causal_logits
 * (attention_eval.cpp:80-91: products rounded, summed in index order, FMA
 * for the < 4-element tail, times scale) and top_k_indices<float> of
 * min(k, n_valid) of them (score desc, index asc; -0 == +0), ascending in
 * idx[p][0..cnt[p]) (row stride k). Bit-identical with the reference.
 * logits (nullable, [P][n_max] f32) receives the logits; NULL uses the
 * context workspace. k == 0 -> SPL_E_DIMENSION ("oracle_topk: k must be >= 1"). */
spl_status spl_oracle_topk(spl_ctx* ctx, const float* q, const void* keys, int kv_dtype,
                           uint64_t cap, uint32_t d, uint32_t P, const uint32_t* n_valid,
                           uint32_t nvalid_div, uint64_t n_max, float scale, uint32_t k,
                           uint32_t* idx, uint32_t* cnt, float* logits, void* stream);
/* matmul (matrix.hpp:81-99) with the reference build's arithmetic (per
 * output, fma over the inner index in order): c[m][n] = a[m][k] . b[k][n],
 * row-major f32. downproj_topk (attention_eval.cpp:183-206) = this for keys
 * and queries, then spl_oracle_topk on the projections with scale 1. */
spl_status spl_project(spl_ctx* ctx, const float* a, uint64_t m, uint32_t k, const float* b,
                       uint32_t n, float* c, void* stream);
/* Generic dense helpers behind the reference's templated host API, for f32
 * and f64 (row-major device arrays). Not on the decode path: the drop-in
 * composes them for matmul<T> (matrix.hpp:81-99) and the double
 * instantiations of mlp_forward / linear_hash / mlp_hash, soft_sign,
 * soft_codes and downproj_scores (hashers.hpp:70-98).
 * spl_matmul: c[m][n] = a[m][k] . b[k][n], each output a fused multiply-add
 * chain over the inner index in order from 0 (the reference build's
 * contraction; bit-exact). k == 0 gives zeros.
 * spl_map: elementwise over x[rows][cols]:
 *   SPL_MAP_BIAS_SILU  out = silu(x + bias[col]), silu(z) = z / (1 + exp(-z))
 *                      (f32: glibc expf port, bit-exact; f64: CUDA exp)
 *   SPL_MAP_SOFT_SIGN  out = gamma x / (1 + gamma |x|), gamma > 0
 *   SPL_MAP_SIGN_BITS  out = u8 (x >= 0), sign(0) -> 1 */
typedef enum spl_map_op {
    SPL_MAP_BIAS_SILU = 0,
    SPL_MAP_SOFT_SIGN = 1,
    SPL_MAP_SIGN_BITS = 2
} spl_map_op;
spl_status spl_matmul(spl_ctx* ctx, int dtype, const void* a, uint64_t m, uint64_t k,
                      const void* b, uint64_t n, void* c, void* stream);
spl_status spl_map(spl_ctx* ctx, int dtype, int op, const void* x, uint64_t rows,
                   uint64_t cols, const void* bias, double gamma, void* out, void* stream);

/* iou (attention_eval.hpp:63, attention_eval.cpp:216-232) per problem of two
 * ascending index lists a[p][0..cnt_a[p]) and b[p][0..cnt_b[p]) (row strides
 * a_stride, b_stride): |a ∩ b| / |a ∪ b| as double, 1.0 when both are empty. */
spl_status spl_iou(spl_ctx* ctx, const uint32_t* a, const uint32_t* cnt_a, uint64_t a_stride,
                   const uint32_t* b, const uint32_t* cnt_b, uint64_t b_stride, uint32_t P,
                   double* out, void* stream);

/* --------------------------------------------------- hamming top-k (K3) */
/* The fused retrieval (hash_topk's hot loop, attention_eval.cpp:172-179:
 * nxor_scores_into(valid) + top_k_indices(min(k, valid))): for every
 * problem p, idx[p][0..cnt[p]) = the min(k, n_valid) rows with the highest
 * agreement with qcodes[p], ties to the lower index, ascending. Bit-exact
 * with the reference. Scores never leave the GPU as int32; n_max (host) is
 * an upper bound of every n_valid used to size the grid. */
spl_status spl_hamming_topk(spl_ctx* ctx, const uint32_t* codes, uint64_t problem_stride_rows,
                            uint32_t L, const uint32_t* qcodes, uint32_t P,
                            const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                            uint32_t k, uint32_t* idx, uint32_t* cnt, void* stream);

/* Sequence-sharded retrieval (SURVEY §8 e), three phases around the caller's
 * collective. Rank r of R owns a contiguous row range of every problem.
 *  1. spl_shard_histogram: local scan; writes hist[p][0..L] (u32 counts of
 *     each agreement score over the local valid rows) and keeps the scores
 *     in the context workspace.
 *  2. caller all-gathers hist from all ranks -> all_hist[R][P][L+1].
 *  3. spl_shard_select: every rank derives the identical global threshold T
 *     and tie quota; rank r keeps score > T plus its share of the score == T
 *     ties (lower ranks first = lower global index first), ascending local
 *     row ids in idx[p][0..cnt[p]), and writes out_offset[p] = the position of
 *     its first index in the global ascending list. The rank-order
 *     concatenation equals the reference's top_k_indices output.
 * k is the GLOBAL budget (min'ed with the global valid count). */
spl_status spl_shard_histogram(spl_ctx* ctx, const uint32_t* codes,
                               uint64_t problem_stride_rows, uint32_t L,
                               const uint32_t* qcodes, uint32_t P, const uint32_t* n_valid,
                               uint32_t nvalid_div, uint64_t n_max, uint32_t* hist,
                               void* stream);
spl_status spl_shard_select(spl_ctx* ctx, const uint32_t* all_hist, uint32_t R, uint32_t rank,
                            uint32_t L, uint32_t P, const uint32_t* n_valid,
                            uint32_t nvalid_div, uint64_t n_max, uint32_t k, uint32_t* idx,
                            uint32_t* cnt, uint32_t* out_offset, void* stream);
/* The host form of step 3's planning arithmetic (same code as the device
 * path), for host-side glue and CPU tests: given all_hist (HOST) for ONE
 * problem, returns T, the global quota of ties, this rank's tie share, the
 * number of indices this rank emits and its offset in the global list. */
spl_status spl_plan_shard_host(const uint32_t* all_hist, uint32_t R, uint32_t rank, uint32_t L,
                               uint32_t k, uint32_t* T, uint32_t* quota, uint32_t* take_eq,
                               uint32_t* count, uint32_t* offset);

/* Fused sequence-sharded retrieval: ONE kernel per rank, the histogram
 * exchange done inside it over peer memory (NVLink P2P stores into every
 * rank's exchange area + release/acquire flags) instead of a host-issued
 * collective between two kernels. Same results as spl_shard_histogram ->
 * all-gather -> spl_shard_select: idx[p][0..cnt[p]) are this rank's local
 * row ids, out_offset[p] their position in the global ascending list, k the
 * GLOBAL budget. Every rank of the group must make the same sequence of
 * calls (they rendezvous inside the kernel; a missing rank turns into
 * SPL_E_CUDA from spl_check_device_error after a 2 s watchdog, not a hang).
 * Setup: spl_peer_create on every rank; exchange the 64-byte handles of
 * spl_peer_ipc_handle (e.g. an all-gather on the host), spl_peer_open with
 * all R handles in rank order. spl_peer_connect_local wires R peers living in
 * ONE process (tests, or several ranks per GPU). L <= 255 (u8 scores) and
 * caches whose scores fit on chip (the fused single-GPU geometry); otherwise
 * SPL_E_STATE and the caller uses the two-kernel flow above. */
typedef struct spl_peer spl_peer;
spl_status spl_peer_create(spl_ctx* ctx, uint32_t R, uint32_t rank, uint32_t P_max,
                           uint32_t L_max, spl_peer** out);
spl_status spl_peer_ipc_handle(spl_ctx* ctx, const spl_peer* peer, void* handle /* host, 64 B */);
spl_status spl_peer_open(spl_ctx* ctx, spl_peer* peer, const void* handles /* host, R x 64 B */);
spl_status spl_peer_connect_local(spl_ctx* ctx, spl_peer* const* peers, uint32_t R);
void spl_peer_destroy(spl_peer* peer);
spl_status spl_hamming_topk_sharded(spl_ctx* ctx, spl_peer* peer, const uint32_t* codes,
                                    uint64_t problem_stride_rows, uint32_t L,
                                    const uint32_t* qcodes, uint32_t P, const uint32_t* n_valid,
                                    uint32_t nvalid_div, uint64_t n_max, uint32_t k,
                                    uint32_t* idx, uint32_t* cnt, uint32_t* out_offset,
                                    void* stream);

/* ------------------------------------------------------ encoders (K1/K2) */
/* A per-head hasher bank (one independent hasher per head).
 * MLP (hashers.hpp:24-34): w1 [H][d][h], b1 [H][h], w2 [H][h][L], row-major
 * f32. LINEAR (hashers.hpp:14-20): w1 = projection [H][d][L], b1/w2 unused
 * (NULL), h = 0. Pointers may be host or device; values are copied. Weights
 * are validated (require_finite, hashers.cpp:90-95 -> SPL_E_NUMERIC). */
spl_status spl_hasher_create(spl_ctx* ctx, int kind, uint32_t H, uint32_t d, uint32_t h,
                             uint32_t L, const float* w1, const float* b1, const float* w2,
                             spl_hasher** out);
void spl_hasher_destroy(spl_hasher* hasher);

/* mlp_forward (hashers.hpp:74-75, hashers.cpp:84-103): pre-activations
 * pre[B][H][m][L] for x[B][H][m][d] (f32), bit-exact with the reference. */
spl_status spl_mlp_forward(spl_ctx* ctx, const spl_hasher* hasher, const float* x, uint32_t B,
                           uint32_t m, float* pre, void* stream);
/* mlp_hash / linear_hash (hashers.hpp:70-79) fused with pack_bits: codes
 * [B][H][m][W]. mode EXACT is bit-exact with the reference; mode TC runs the
 * tcgen05 bulk encoder (bits may differ only where |pre-activation| lies in
 * the bf16 error band). Non-finite input raises the device error word. */
spl_status spl_encode(spl_ctx* ctx, const spl_hasher* hasher, const float* x, uint32_t B,
                      uint32_t m, int mode, uint32_t* codes, void* stream);
/* Bulk / prefill encode on the tcgen05 tensor cores (K2, the SPL_ENCODE_TC
 * mode of spl_encode with a choice of input dtype): x [B][H][m][d] f32 or
 * bf16 (x_dtype SPL_F32 / SPL_BF16) -> codes [B][H][m][W]; bf16 operands,
 * fp32 accumulation. Needs d = 128 (MLP: h = 128) and L in {32, 64, 128,
 * 256}, else SPL_E_DIMENSION. pre (nullable) receives the f32
 * pre-activations [B][H][m][L] (numerics tests). Replaces the same
 * mlp_hash / linear_hash + pack_bits as spl_encode (hashers.hpp:70-79). */
spl_status spl_encode_tc(spl_ctx* ctx, const spl_hasher* hasher, const void* x, int x_dtype,
                         uint32_t B, uint32_t m, uint32_t* codes, float* pre, void* stream);
/* Decode-time append (new capability): for every (b, head),
 * encode k_new[b][head] (exact mode) into codes[b][head][pos[b]] and copy
 * k_new / v_new into the K/V caches at the same slot (kv_dtype storage,
 * [B][H][cap][d]). pos is a device array [B]. */
spl_status spl_encode_append(spl_ctx* ctx, const spl_hasher* hasher, const float* k_new,
                             const float* v_new, uint32_t B, uint32_t* codes, void* kcache,
                             void* vcache, int kv_dtype, uint64_t cap, const uint32_t* pos,
                             void* stream);

/* ----------------------------------------------- sparse attention (K4/K5) */
/* sparse_attention (attention_eval.hpp:67, attention_eval.cpp:234-264 with
 * attend_subset :54-78): for every problem p, softmax(q K_S^T * scale) V_S
 * over S = idx[p][0..cnt[p]) U {n_valid - 1} (own token always attended),
 * fp32 accumulation, flash-decoding split + log-sum-exp combine.
 * q/out: [P][d] f32; kcache/vcache rows at base + p*problem_stride_rows*d.
 * Indices must be < n_valid (the reference's DimensionError check is done
 * by the C++ drop-in on the host). */
spl_status spl_sparse_attend(spl_ctx* ctx, const float* q, const void* kcache,
                             const void* vcache, int kv_dtype, uint64_t problem_stride_rows,
                             uint32_t d, uint32_t P, const uint32_t* idx, uint64_t idx_stride,
                             const uint32_t* cnt, const uint32_t* n_valid, uint32_t nvalid_div,
                             float scale, float* out, void* stream);
/* Sharded form: partials[p] = (m, l, o[d]) over this rank's rows only
 * (own token included only when include_own != 0), then
 * spl_attend_combine merges R gathered partial sets [R][P][d+2]. */
spl_status spl_sparse_attend_partial(spl_ctx* ctx, const float* q, const void* kcache,
                                     const void* vcache, int kv_dtype,
                                     uint64_t problem_stride_rows, uint32_t d, uint32_t P,
                                     const uint32_t* idx, uint64_t idx_stride,
                                     const uint32_t* cnt, const uint32_t* own_row,
                                     uint32_t nvalid_div, float scale, float* partials,
                                     void* stream);
spl_status spl_attend_combine(spl_ctx* ctx, const float* partials, uint32_t R, uint32_t P,
                              uint32_t d, float* out, void* stream);

/* --------------------------------------------------------- decode step */
/* One decode step of one layer for B sequences x H heads:
 *   append: codes/K/V[b][h][n_valid[b]-1] <- encode(k_new), k_new, v_new
 *   encode: qcodes <- encode(q)                       (exact mode)
 *   retrieve: idx/cnt <- hamming top-k(min(k, n_valid))
 *   attend: out <- sparse attention over idx U {own}
 * All arrays device; idx [B*H][k], cnt [B*H], out [B][H][d]. */
spl_status spl_decode_step(spl_ctx* ctx, const spl_hasher* hasher, const float* q,
                           const float* k_new, const float* v_new, uint32_t B,
                           uint32_t* codes, void* kcache, void* vcache, int kv_dtype,
                           uint64_t cap, const uint32_t* n_valid, uint64_t n_max, uint32_t k,
                           float scale, uint32_t* idx, uint32_t* cnt, float* out, void* stream);

/* One decode step of one layer on ONE RANK of a sequence-sharded KV cache
 * (SURVEY §8 e, config 5): every rank holds a contiguous slice of each
 * sequence's tokens (codes/K/V [B][H][cap][.], its local n_valid[B]); the
 * step's new token belongs to exactly one rank (owner != 0 there, e.g. the
 * last rank), which appends it at its local n_valid[b] - 1 — the own token
 * sparse_attention always attends (attention_eval.cpp:249-260).
 *   every rank: encode q; retrieval of the GLOBAL top-k (k = the global
 *   budget) with the histogram exchange inside the kernel over peer memory;
 *   partial attention over its own selected rows; exchange of the (m, l, o)
 *   partials, again inside the kernel; log-sum-exp combine.
 * idx/cnt/out_offset: this rank's share of the reference's index list (as
 * spl_hamming_topk_sharded: local ids, position in the global list);
 * out [B][H][d]: the full attention output, identical on every rank.
 * All ranks of the peer group must make the same sequence of calls. One
 * launch after the encoder when L = d = 128 and the local scores fit on
 * chip; otherwise sharded retrieval + partial attention + peer combine. */
spl_status spl_sharded_decode_step(spl_ctx* ctx, spl_peer* peer, const spl_hasher* hasher,
                                   const float* q, const float* k_new, const float* v_new,
                                   uint32_t B, int owner, uint32_t* codes, void* kcache,
                                   void* vcache, int kv_dtype, uint64_t cap,
                                   const uint32_t* n_valid, uint64_t n_max, uint32_t k, float scale,
                                   uint32_t* idx, uint32_t* cnt, uint32_t* out_offset, float* out,
                                   void* stream);

/* budget_from_rate (attention_eval.hpp:70, attention_eval.cpp:266-272). */
spl_status spl_budget_from_rate(double rate, uint64_t n, uint32_t* k);

/* ---------------------------------------------------------------- training
 * Hasher training. Mirrors spotlight::train_hasher
 * (trainer.hpp:115-118, trainer.cpp:634-645): RankingLossConfig
 * (ranking_loss.hpp:15-24; optional counts < 0 = unset) and TrainConfig
 * (trainer.hpp:18-37); loss_kind = TrainLoss (trainer.hpp:82). */
typedef struct spl_rank_config {
    double beta, alpha, maskout;
    int64_t max_top, max_oth, query_subsample; /* < 0: unset (std::nullopt) */
} spl_rank_config;
typedef struct spl_train_config {
    uint32_t num_iters, warmup_iters, batch, holdout_queries;
    uint64_t seed;
    double max_lr, min_lr, adam_beta1, adam_beta2, adam_eps, weight_decay, grad_clip,
        soft_gamma, holdout_budget_rate;
} spl_train_config;
/* All pointers HOST. kind: SPL_HASHER_MLP (w1 d x h, b1 h, w2 h x L, gamma =
 * the hasher's), SPL_HASHER_LINEAR (w1 = projection d x L, soft_gamma) or
 * SPL_HASHER_DOWNPROJ (w1 = projection d x L). Weights are updated in place
 * (also when an error stops the run, as the reference's in-place hasher).
 * Sequences are concatenated: sequence s has seq_len[s] query rows and as
 * many key rows (causally aligned). records: [num_iters][3] = {loss,
 * violation_rate, lr} (IterRecord, trainer.hpp:84-89). Per-row orders are
 * sorted in shared-memory chunks of 16384 keys, merged in global memory
 * beyond that.
 * Limits the reference does not have (it streams each query): the sampled
 * top + other keys per query must be <= 12800 (one block's shared memory),
 * and the pair gradients (queries x top x other doubles) must fit in half
 * the free device memory; beyond either, SPL_E_DIMENSION ("GPU trainer
 * limit: ...") — set max_top / max_oth / query_subsample, as the CLI does. */
typedef enum spl_train_loss {
    SPL_TRAIN_LOSS_RANKING = 0,        /* TrainLoss::ranking */
    SPL_TRAIN_LOSS_RECONSTRUCTION = 1  /* TrainLoss::reconstruction (MSE ablation) */
} spl_train_loss;
spl_status spl_train_hasher(spl_ctx* ctx, int kind, uint32_t d, uint32_t h, uint32_t L,
                            float gamma, float* w1, float* b1, float* w2, uint32_t n_seq,
                            const float* queries, const float* keys, const uint32_t* seq_len,
                            const spl_rank_config* rank, const spl_train_config* train,
                            int loss_kind, double* records, double* holdout_iou,
                            uint32_t* skipped, void* stream);
/* partition_topk's draws (ranking_loss.cpp:80-116), host only: rows
 * [min(query_subsample, q_train)], top positions [min(max_top, k_full)], other
 * positions relative to k_full [min(max_oth, n - k_full)]; counts = {rows,
 * top, other, k_full}. */
spl_status spl_train_partition_host(const spl_rank_config* rank, uint32_t q_train, uint32_t n,
                                    uint64_t seed, uint32_t* rows, uint32_t* top_pos,
                                    uint32_t* oth_pos, uint32_t* counts);
/* Device time (CUDA events) of the iteration loop of the last
 * spl_train_hasher call on this context, ms (setup and holdout excluded). */
double spl_train_last_loop_ms(const spl_ctx* ctx);
/* lr_at (trainer.cpp:35-46) */
double spl_train_lr_at(uint32_t iter, const spl_train_config* train);

#ifdef __cplusplus
}
#endif
#endif /* SPL_C_H */
