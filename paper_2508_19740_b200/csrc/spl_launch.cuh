// Launch-level interfaces shared between the kernel files and capi.cu.
#pragma once
#include "spl_internal.cuh"

namespace spl {

enum EncOut { ENC_CODES = 0, ENC_PRE = 1, ENC_APPEND = 2 };

struct EncJob {
    const float* x;       // [B][H][m][d]
    uint32_t m;
    int out_mode;
    uint32_t* codes;      // ENC_CODES: [B][H][m][W]; ENC_APPEND: [B][H][cap][W]
    float* pre;           // ENC_PRE: [B][H][m][L]
    uint64_t cap;
    const uint32_t* pos;  // ENC_APPEND: slot per batch (pos[b] - pos_minus_one)
    int pos_minus_one;    // 1: pos holds n_valid (slot = n_valid - 1)
    const float* v_new;   // ENC_APPEND: copy k/v rows into the caches
    void* kcache;
    void* vcache;
    int kv_dtype;
};

struct AttParams {
    const float* q;
    const void* kc;
    const void* vc;
    uint64_t stride_rows;
    uint32_t d;
    uint32_t P;
    const uint32_t* idx;
    uint64_t idx_stride;
    const uint32_t* cnt;
    const uint32_t* n_valid;   // own = n_valid[p / div] - 1   (normal mode)
    const uint32_t* own_row;   // own row per problem, ~0u = none (partial mode)
    uint32_t nvalid_div;
    float qscale;              // scale * log2(e)
    uint32_t rows_per_split;
    uint32_t nsplit;
    float* partials;           // [P][nsplit][d + 2]
    uint32_t* counters;        // [P]
    float* out;                // normal: [P][d]; partial mode: [P][d + 2] (m, l, o)
    int partial_mode;
    int own_nvalid;            // partial mode: own = n_valid[p / div] - 1 (own_row unused)
};

// hamming_topk.cu
spl_status hamming_topk_impl(spl_ctx*, const uint32_t*, uint64_t, uint32_t, const uint32_t*,
                             uint32_t, const uint32_t*, uint32_t, uint64_t, uint32_t, uint32_t*,
                             uint32_t*, cudaStream_t);
spl_status hamming_topk_attend_impl(spl_ctx*, const uint32_t*, uint64_t, uint32_t,
                                    const uint32_t*, uint32_t, const uint32_t*, uint32_t, uint64_t,
                                    uint32_t, uint32_t*, uint32_t*, const float*, const void*,
                                    const void*, int, uint32_t, float, float*, cudaStream_t, bool*,
                                    spl_peer* = nullptr, uint32_t* = nullptr, int = 1);
spl_status peer_combine_launch(spl_ctx*, spl_peer*, const float*, uint32_t, uint32_t, float*,
                               cudaStream_t);
spl_status shard_histogram_impl(spl_ctx*, const uint32_t*, uint64_t, uint32_t, const uint32_t*,
                                uint32_t, const uint32_t*, uint32_t, uint64_t, uint32_t*,
                                cudaStream_t);
spl_status shard_select_impl(spl_ctx*, const uint32_t*, uint32_t, uint32_t, uint32_t, uint32_t,
                             const uint32_t*, uint32_t, uint64_t, uint32_t, uint32_t*, uint32_t*,
                             uint32_t*, cudaStream_t);
spl_status hamming_topk_sharded_impl(spl_ctx*, spl_peer*, const uint32_t*, uint64_t, uint32_t,
                                     const uint32_t*, uint32_t, const uint32_t*, uint32_t,
                                     uint64_t, uint32_t, uint32_t*, uint32_t*, uint32_t*,
                                     cudaStream_t);
uint64_t peer_area_words(uint32_t R, uint32_t Pmax, uint32_t Lmax);
// lazy-module preloads (spl_peer_create): encoder, K4 / K5, sharded K3
void encode_preload();
void attend_preload();
void k3_preload();
// bitcodes_misc.cu
spl_status pack_bits_launch(spl_ctx*, const uint8_t*, uint64_t, uint32_t, uint32_t*, cudaStream_t);
spl_status unpack_bits_launch(spl_ctx*, const uint32_t*, uint64_t, uint32_t, uint8_t*,
                              cudaStream_t);
spl_status nxor_scores_launch(spl_ctx*, const uint32_t*, uint64_t, uint32_t, const uint32_t*,
                              uint32_t, const uint32_t*, uint32_t, uint64_t, int32_t*, uint64_t,
                              cudaStream_t);
spl_status top_k_launch(spl_ctx*, const void*, int, uint32_t, uint64_t, uint64_t, uint32_t,
                        uint32_t*, cudaStream_t, const uint32_t* n_valid = nullptr,
                        uint32_t nvalid_div = 1, uint32_t* cnt = nullptr);
// dense_retrieval.cu
spl_status causal_logits_launch(spl_ctx*, const float* q, const void* keys, int kv_dtype,
                                uint64_t cap, uint32_t d, uint32_t P, const uint32_t* n_valid,
                                uint32_t nvalid_div, uint64_t n_max, float scale, float* logits,
                                cudaStream_t);
spl_status project_launch(spl_ctx*, const float* a, uint64_t m, uint32_t k, const float* b,
                          uint32_t n, float* c, cudaStream_t);
spl_status iou_launch(spl_ctx*, const uint32_t* a, const uint32_t* cnt_a, uint64_t a_stride,
                      const uint32_t* b, const uint32_t* cnt_b, uint64_t b_stride, uint32_t P,
                      double* out, cudaStream_t);
// encode_exact.cu
spl_status encode_exact_launch(spl_ctx*, const spl_hasher*, uint32_t, const EncJob*, int,
                               cudaStream_t);
// encode_tc.cu
spl_status encode_tc_launch(spl_ctx*, const spl_hasher*, const void* x, int x_dtype, uint32_t B,
                            uint32_t m, uint32_t* codes, float* pre, cudaStream_t);
bool encode_tc_eligible(uint32_t kind, uint32_t d, uint32_t h, uint32_t L);
// sparse_attend.cu
spl_status sparse_attend_launch(spl_ctx*, AttParams, uint32_t, int, cudaStream_t);
uint32_t att_rows_per_split();  // list entries per K4 CTA (sizes the partials)
spl_status sparse_attend_reserve(spl_ctx*, uint32_t P, uint32_t kmax, uint32_t d, cudaStream_t);
spl_status attend_combine_launch(spl_ctx*, const float*, uint32_t, uint32_t, uint32_t, float*,
                                 cudaStream_t);

}  // namespace spl
