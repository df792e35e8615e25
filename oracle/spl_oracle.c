/* TEST INFRASTRUCTURE ONLY — see spl_oracle.h. Plain-C restatement of the
 * reference's hot path. Built with -ffp-contract=off: every fused
 * multiply-add that GCC contracts in the reference build (-march=native =>
 * -ffp-contract=fast, confirmed by vfmadd in hashers.o) is written here as an
 * explicit fmaf(), every other operation is a separately rounded float op, and
 * exp is glibc's expf, the very libm routine the reference calls. */
#include "spl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ bitcodes */

/* bitcodes.cpp:22-41: for chunk c = 0..31, word <<= 1, |= column c*cw + w. */
int orc_pack_bits(const uint8_t* bits, uint32_t n, uint32_t d, uint32_t* words) {
    if (d == 0 || d % 32 != 0) return 1;
    const uint32_t cw = d / 32;
    for (uint32_t i = 0; i < n; ++i) {
        const uint8_t* brow = bits + (size_t)i * d;
        uint32_t* orow = words + (size_t)i * cw;
        for (uint32_t w = 0; w < cw; ++w) orow[w] = 0;
        for (uint32_t c = 0; c < 32; ++c)
            for (uint32_t w = 0; w < cw; ++w)
                orow[w] = (orow[w] << 1) | (uint32_t)(brow[c * cw + w] & 1u);
    }
    return 0;
}

/* bitcodes.cpp:43-57. */
int orc_unpack_bits(const uint32_t* words, uint32_t n, uint32_t L, uint8_t* bits) {
    if (L == 0 || L % 32 != 0) return 1;
    const uint32_t cw = L / 32;
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t w = 0; w < cw; ++w) {
            const uint32_t word = words[(size_t)i * cw + w];
            for (uint32_t c = 0; c < 32; ++c)
                bits[(size_t)i * L + c * cw + w] = (uint8_t)((word >> (31 - c)) & 1u);
        }
    return 0;
}

/* bitcodes.cpp:59-76: agree += popcount(~(q ^ r)) over words. The length
 * check (:62-65) raises DimensionError. */
int orc_nxor_scores_into(const uint32_t* q, uint32_t q_words, const uint32_t* words,
                         uint32_t n, uint32_t L, uint32_t n_valid, int32_t* out) {
    const uint32_t W = L / 32;
    (void)n;
    if (q_words != W) return 1;
    for (uint32_t i = 0; i < n_valid; ++i) {
        const uint32_t* r = words + (size_t)i * W;
        int32_t agree = 0;
        for (uint32_t w = 0; w < W; ++w) agree += __builtin_popcount(~(q[w] ^ r[w]));
        out[i] = agree;
    }
    return 0;
}

/* bitcodes.cpp:89-131. Entry + ranks_ahead (:91-104): a ranks ahead of b if
 * it has the higher score, or the same score and the lower index. The heap
 * keeps the k best with the current worst at its root (:114-126); the kept
 * indices are returned sorted ascending (:127-129). */
typedef struct { double s; uint32_t idx; } orc_entry;

static int ranks_ahead(const orc_entry* a, const orc_entry* b) {
    if (a->s != b->s) return a->s > b->s;
    return a->idx < b->idx;
}

/* Max-heap w.r.t. "ranks behind": root = the entry every other entry ranks
 * ahead of (std::push_heap/pop_heap with comparator ranks_ahead). */
static void heap_up(orc_entry* h, size_t i) {
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (ranks_ahead(&h[p], &h[i])) {
            orc_entry t = h[p]; h[p] = h[i]; h[i] = t; i = p;
        } else break;
    }
}
static void heap_down(orc_entry* h, size_t n, size_t i) {
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && ranks_ahead(&h[m], &h[l])) m = l;
        if (r < n && ranks_ahead(&h[m], &h[r])) m = r;
        if (m == i) break;
        orc_entry t = h[m]; h[m] = h[i]; h[i] = t; i = m;
    }
}
static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

static int top_k_generic(const void* scores, int is_float, uint32_t n, uint32_t k,
                         uint32_t* out) {
    if (k == 0 || k > n) return 1; /* bitcodes.cpp:110-113 */
    orc_entry* heap = (orc_entry*)malloc(sizeof(orc_entry) * k);
    size_t size = 0;
    for (uint32_t i = 0; i < n; ++i) {
        orc_entry cand;
        cand.s = is_float ? (double)((const float*)scores)[i] : (double)((const int32_t*)scores)[i];
        cand.idx = i;
        if (size < k) {
            heap[size++] = cand;
            heap_up(heap, size - 1);
        } else if (ranks_ahead(&cand, &heap[0])) {
            heap[0] = cand;
            heap_down(heap, size, 0);
        }
    }
    for (size_t i = 0; i < size; ++i) out[i] = heap[i].idx;
    qsort(out, size, sizeof(uint32_t), cmp_u32);
    free(heap);
    return 0;
}

int orc_top_k_i32(const int32_t* scores, uint32_t n, uint32_t k, uint32_t* out) {
    return top_k_generic(scores, 0, n, k, out);
}
int orc_top_k_f32(const float* scores, uint32_t n, uint32_t k, uint32_t* out) {
    return top_k_generic(scores, 1, n, k, out);
}

/* ------------------------------------------------------------- hashers */

static int all_finite(const float* p, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(p[i])) return 0;
    return 1;
}

/* matrix.hpp:81-99: c[i][j] starts at 0 and, for p = 0..k-1 in order,
 * c[i][j] += a[i][p] * b[p][j] — contracted to one FMA per step. */
static void matmul_fma(const float* a, const float* b, float* c, uint32_t m, uint32_t k,
                       uint32_t n) {
    for (uint32_t i = 0; i < m; ++i) {
        float* crow = c + (size_t)i * n;
        for (uint32_t j = 0; j < n; ++j) crow[j] = 0.0f;
        for (uint32_t p = 0; p < k; ++p) {
            const float av = a[(size_t)i * k + p];
            const float* brow = b + (size_t)p * n;
            for (uint32_t j = 0; j < n; ++j) crow[j] = fmaf(av, brow[j], crow[j]);
        }
    }
}

/* hashers.cpp:30-33: z / (1 + exp(-z)), every op rounded in float. */
static float silu(float z) {
    const float e = expf(-z);
    const float den = 1.0f + e;
    return z / den;
}

/* hashers.cpp:84-103. require_finite (:14-17) order: w1, w2, b1, input. */
int orc_mlp_forward(const float* w1, const float* b1, const float* w2, uint32_t d, uint32_t h,
                    uint32_t L, const float* x, uint32_t m, float* pre) {
    if (!all_finite(w1, (size_t)d * h) || !all_finite(w2, (size_t)h * L) ||
        !all_finite(b1, h) || !all_finite(x, (size_t)m * d))
        return 2;
    float* z1 = (float*)malloc(sizeof(float) * (size_t)m * h);
    matmul_fma(x, w1, z1, m, d, h);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < h; ++j) {
            const float z = z1[i * h + j] + b1[j];
            z1[i * h + j] = silu(z);
        }
    matmul_fma(z1, w2, pre, m, h, L);
    free(z1);
    return 0;
}

/* sign_bits (hashers.cpp:19-28): bit = (pre >= 0), so -0.0 and +0.0 -> 1. */
static void sign_pack(const float* pre, uint32_t m, uint32_t L, uint32_t* codes) {
    uint8_t* bits = (uint8_t*)malloc((size_t)m * L);
    for (size_t i = 0; i < (size_t)m * L; ++i) bits[i] = pre[i] >= 0.0f;
    orc_pack_bits(bits, m, L, codes);
    free(bits);
}

int orc_mlp_hash_packed(const float* w1, const float* b1, const float* w2, uint32_t d,
                        uint32_t h, uint32_t L, const float* x, uint32_t m, uint32_t* codes) {
    if (L == 0 || L % 32 != 0) return 1;
    float* pre = (float*)malloc(sizeof(float) * (size_t)m * L);
    int st = orc_mlp_forward(w1, b1, w2, d, h, L, x, m, pre);
    if (st == 0) sign_pack(pre, m, L, codes);
    free(pre);
    return st;
}

/* hashers.cpp:75-82: sign(x * projection). No finiteness check there. */
int orc_linear_hash_packed(const float* proj, uint32_t d, uint32_t L, const float* x,
                           uint32_t m, uint32_t* codes) {
    if (L == 0 || L % 32 != 0) return 1;
    float* pre = (float*)malloc(sizeof(float) * (size_t)m * L);
    matmul_fma(x, proj, pre, m, d, L);
    sign_pack(pre, m, L, codes);
    free(pre);
    return 0;
}

/* ------------------------------------------------------ attention_eval */

/* attention_eval.cpp:266-272. */
uint32_t orc_budget_from_rate(double rate, uint64_t n, int* status) {
    *status = 0;
    if (!(rate > 0.0 && rate <= 1.0)) {
        *status = 1;
        return 0;
    }
    uint32_t raw = (uint32_t)(rate * (double)n);
    uint64_t k = raw > 20 ? raw : 20;
    return (uint32_t)(k < n ? k : n);
}

/* The logit dot product of attend_subset (attention_eval.cpp:61-63,
 * `acc += q[p] * krow[p]`) as the reference build compiles it: GCC
 * vectorises the products of this in-order float reduction (8-wide main
 * loop, then a 4-wide epilogue — vmulps + sequential vaddss, so those
 * products are rounded before the add) and contracts only the scalar tail
 * (< 4 elements, vfmadd231ss). The accumulation ORDER is the source order
 * throughout; only the rounding of the product differs by position. */
static float ref_dot(const float* q, const float* k, uint32_t d) {
    float acc = 0.0f;
    uint32_t p = 0;
    const uint32_t n8 = d / 8 * 8;
    for (; p < n8; ++p) acc = acc + q[p] * k[p];
    if (d - p >= 4)
        for (uint32_t e = p + 4; p < e; ++p) acc = acc + q[p] * k[p];
    for (; p < d; ++p) acc = fmaf(q[p], k[p], acc);
    return acc;
}

/* causal_logits (attention_eval.cpp:80-91): the same `acc += q[p] * k[p]`
 * loop as attend_subset, compiled the same way (ref_dot), times scale.
 * oracle_topk (attention_eval.cpp:121-135): per query, top_k_indices<float>
 * over its causal logits with k clamped to the causal range. out[i][k]
 * holds min(k, offsets[i]) ascending indices; counts[i] that number. */
int orc_oracle_topk(const float* queries, uint32_t q, const float* keys, uint32_t n, uint32_t d,
                    float scale, const uint32_t* offsets, uint32_t k, uint32_t* out,
                    uint32_t* counts) {
    if (k == 0) return 1;
    float* logits = (float*)malloc(sizeof(float) * (n ? n : 1));
    if (!logits) return 1;
    for (uint32_t i = 0; i < q; ++i) {
        const uint32_t valid = offsets[i];
        if (valid == 0 || valid > n) {
            free(logits);
            return 1;
        }
        for (uint32_t j = 0; j < valid; ++j)
            logits[j] = ref_dot(queries + (size_t)i * d, keys + (size_t)j * d, d) * scale;
        const uint32_t kk = k < valid ? k : valid;
        counts[i] = kk;
        if (orc_top_k_f32(logits, valid, kk, out + (size_t)i * k)) {
            free(logits);
            return 1;
        }
    }
    free(logits);
    return 0;
}

/* attend_subset, attention_eval.cpp:54-78. */
static void attend_subset(const float* q, const float* keys, const float* values, uint32_t d,
                          float scale, const uint32_t* idx, size_t cnt, float* out) {
    float* logits = (float*)malloc(sizeof(float) * (cnt ? cnt : 1));
    float mx = -INFINITY;
    for (size_t j = 0; j < cnt; ++j) {
        const float* k = keys + (size_t)idx[j] * d;
        const float acc = ref_dot(q, k, d);
        logits[j] = acc * scale;
        mx = (mx < logits[j]) ? logits[j] : mx; /* std::max(max_logit, l) */
    }
    for (uint32_t p = 0; p < d; ++p) out[p] = 0.0f;
    float denom = 0.0f;
    for (size_t j = 0; j < cnt; ++j) {
        const float w = expf(logits[j] - mx);
        denom += w;
        const float* v = values + (size_t)idx[j] * d;
        for (uint32_t p = 0; p < d; ++p) out[p] = fmaf(w, v[p], out[p]);
    }
    const float inv = 1.0f / denom;
    for (uint32_t p = 0; p < d; ++p) out[p] *= inv;
    free(logits);
}

/* attention_eval.cpp:234-264 (validate :13-30): picked must be non-empty and
 * inside the causal range; the own row (offset - 1) is always inserted. */
int orc_sparse_attention(const float* queries, uint32_t q, const float* keys,
                         const float* values, uint32_t n, uint32_t d, float scale,
                         const uint32_t* offsets, const uint32_t* picked,
                         const uint64_t* picked_off, float* out) {
    if (n == 0 || !(scale > 0.0f)) return 1;
    for (uint32_t r = 0; r < q; ++r)
        if (offsets[r] == 0 || offsets[r] > n) return 1;
    for (uint32_t r = 0; r < q; ++r) {
        const uint64_t b = picked_off[r], e = picked_off[r + 1];
        if (e == b) return 1;
        const uint32_t valid = offsets[r], own = valid - 1;
        size_t cnt = (size_t)(e - b);
        uint32_t* sub = (uint32_t*)malloc(sizeof(uint32_t) * (cnt + 1));
        int has_own = 0;
        for (size_t j = 0; j < cnt; ++j) {
            sub[j] = picked[b + j];
            if (sub[j] >= valid) { free(sub); return 1; }
            if (sub[j] == own) has_own = 1;
        }
        if (!has_own) { /* insert at upper_bound (the picked list is sorted) */
            size_t pos = cnt;
            while (pos > 0 && sub[pos - 1] > own) { sub[pos] = sub[pos - 1]; --pos; }
            sub[pos] = own;
            ++cnt;
        }
        attend_subset(queries + (size_t)r * d, keys, values, d, scale, sub, cnt,
                      out + (size_t)r * d);
        free(sub);
    }
    return 0;
}

/* attention_eval.cpp:172-179 per problem, over P problems. */
int orc_retrieve_batch(const uint32_t* codes, uint32_t P, uint64_t cap, uint32_t L,
                       const uint32_t* qcodes, const uint32_t* n_valid, uint32_t k,
                       uint32_t* out, int threads) {
    const uint32_t W = L / 32;
    int status = 0;
    if (k == 0) return 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
    for (uint32_t p = 0; p < P; ++p) {
        const uint32_t n = n_valid[p];
        int32_t* scores = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
        int st = orc_nxor_scores_into(qcodes + (size_t)p * W, W, codes + (size_t)p * cap * W,
                                      n, L, n, scores);
        if (st == 0) st = orc_top_k_i32(scores, n, k < n ? k : n, out + (size_t)p * k);
        if (st) {
#pragma omp atomic write
            status = st;
        }
        free(scores);
    }
    return status;
}
