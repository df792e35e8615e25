// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libspotref.so, namespace renamed spotlight -> spotref).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg load it: it is the checker and the CPU baseline,
// never the thing measured as the product.
//
// Every entry point returns 0 on success, or a nonzero code with the
// reference exception's what() copied into spotref_last_error():
//   1 DimensionError, 2 NumericError, 3 FormatError, 4 IoError, 9 other.

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "spotlight/attention_eval.hpp"
#include "spotlight/bitcodes.hpp"
#include "spotlight/errors.hpp"
#include "spotlight/hashers.hpp"
#include "spotlight/linalg.hpp"
#include "spotlight/rng.hpp"
#include "spotlight/ranking_loss.hpp"
#include "spotlight/trainer.hpp"

using namespace spotlight;  // == spotref under -Dspotlight=spotref

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 1;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const EmptyPairError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

Matrix<float> mat(const float* p, std::size_t r, std::size_t c) {
    return Matrix<float>(r, c, std::vector<float>(p, p + r * c));
}

MlpHasher make_mlp(const float* w1, const float* b1, const float* w2, std::uint32_t d,
                   std::uint32_t h, std::uint32_t L) {
    MlpHasher m;
    m.w1 = mat(w1, d, h);
    m.b1.assign(b1, b1 + h);
    m.w2 = mat(w2, h, L);
    m.gamma = 64.0f;
    return m;
}

CodeMatrix codes_from(const std::uint32_t* words, std::uint32_t n, std::uint32_t L) {
    CodeMatrix c(n, L);
    std::memcpy(c.raw().data(), words, sizeof(std::uint32_t) * n * (L / 32));
    return c;
}

void copy_bits(const BitMatrix& b, std::uint8_t* out) {
    for (std::size_t i = 0; i < b.rows(); ++i) {
        const auto r = b.row(i);
        std::memcpy(out + i * b.cols(), r.data(), b.cols());
    }
}
}  // namespace

extern "C" {

const char* spotref_last_error() { return g_err.c_str(); }

int spotref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

std::uint64_t spotref_derive_seed(std::uint64_t base, std::uint64_t stream) {
    return derive_seed(base, stream);
}

// mlp_gaussian_init (hashers.cpp:41-63).
int spotref_mlp_gaussian_init(std::uint32_t d, std::uint32_t h, std::uint32_t L, float gamma,
                              std::uint64_t seed, float* w1, float* b1, float* w2) {
    return guard([&] {
        const MlpHasher m = mlp_gaussian_init(d, h, L, gamma, seed);
        std::memcpy(w1, m.w1.data(), sizeof(float) * m.w1.size());
        std::memcpy(b1, m.b1.data(), sizeof(float) * m.b1.size());
        std::memcpy(w2, m.w2.data(), sizeof(float) * m.w2.size());
    });
}

// qr_rotation_init (hashers.cpp:37-39) -> d x d projection.
int spotref_qr_rotation_init(std::uint32_t d, std::uint64_t seed, float* proj) {
    return guard([&] {
        const LinearHasher l = qr_rotation_init(d, seed);
        std::memcpy(proj, l.projection.data(), sizeof(float) * l.projection.size());
    });
}

// downproj_init (hashers.cpp:65-74) -> d x r projection.
int spotref_downproj_init(std::uint32_t d, std::uint32_t r, std::uint64_t seed, float* proj) {
    return guard([&] {
        const DownProjEstimator e = downproj_init(d, r, seed);
        std::memcpy(proj, e.projection.data(), sizeof(float) * e.projection.size());
    });
}

// random_rotation (linalg.cpp:80-92), f64 d x d.
int spotref_random_rotation(std::uint32_t d, std::uint64_t seed, double* q) {
    return guard([&] {
        const Matrix<double> m = random_rotation(d, seed);
        std::memcpy(q, m.data(), sizeof(double) * m.size());
    });
}

// write_hasher (hashers.cpp:184-215): kind 0 linear (w1 = d x L projection),
// 1 mlp (w1 d x h, b1 h, w2 h x L, gamma), 2 downproj (w1 = d x L).
int spotref_write_hasher(const char* path, int kind, std::uint32_t d, std::uint32_t h,
                         std::uint32_t L, float gamma, const float* w1, const float* b1,
                         const float* w2) {
    return guard([&] {
        if (kind == 1) {
            MlpHasher m = make_mlp(w1, b1, w2, d, h, L);
            m.gamma = gamma;
            write_hasher(path, AnyHasher{m});
        } else if (kind == 0) {
            write_hasher(path, AnyHasher{LinearHasher{mat(w1, d, L)}});
        } else {
            write_hasher(path, AnyHasher{DownProjEstimator{mat(w1, d, L)}});
        }
    });
}

// read_hasher (hashers.cpp:217-246): dims[4] = {kind, d, h, L}; the
// parameter buffers (may be null on a first call that only asks for dims)
// are filled when non-null.
int spotref_read_hasher(const char* path, std::uint32_t* dims, float* gamma, float* w1, float* b1,
                        float* w2) {
    return guard([&] {
        const AnyHasher a = read_hasher(path);
        if (const auto* m = std::get_if<MlpHasher>(&a)) {
            dims[0] = 1;
            dims[1] = m->input_dim();
            dims[2] = m->hidden_dim();
            dims[3] = m->code_bits();
            *gamma = m->gamma;
            if (w1) std::memcpy(w1, m->w1.data(), sizeof(float) * m->w1.size());
            if (b1) std::memcpy(b1, m->b1.data(), sizeof(float) * m->b1.size());
            if (w2) std::memcpy(w2, m->w2.data(), sizeof(float) * m->w2.size());
        } else {
            const Matrix<float>& p = std::holds_alternative<LinearHasher>(a)
                                         ? std::get<LinearHasher>(a).projection
                                         : std::get<DownProjEstimator>(a).projection;
            dims[0] = std::holds_alternative<LinearHasher>(a) ? 0 : 2;
            dims[1] = (std::uint32_t)p.rows();
            dims[2] = 0;
            dims[3] = (std::uint32_t)p.cols();
            *gamma = 0.0f;
            if (w1) std::memcpy(w1, p.data(), sizeof(float) * p.size());
        }
    });
}

// write_code_index / read_code_index (bitcodes.cpp:138-160), SPLC.
int spotref_write_code_index(const char* path, const std::uint32_t* words, std::uint32_t n,
                             std::uint32_t L) {
    return guard([&] { write_code_index(path, codes_from(words, n, L)); });
}
int spotref_read_code_index(const char* path, std::uint32_t* n, std::uint32_t* L,
                            std::uint32_t* words) {
    return guard([&] {
        const CodeMatrix c = read_code_index(path);
        *n = c.rows();
        *L = c.length_bits();
        if (words) std::memcpy(words, c.raw().data(), sizeof(std::uint32_t) * c.raw().size());
    });
}

// pack_bits (bitcodes.cpp:22-41): bits[n][d] bytes -> words[n][d/32].
int spotref_pack_bits(const std::uint8_t* bits, std::uint32_t n, std::uint32_t d,
                      std::uint32_t* words) {
    return guard([&] {
        BitMatrix b(n, d);
        for (std::uint32_t i = 0; i < n; ++i)
            for (std::uint32_t j = 0; j < d; ++j) b.set(i, j, bits[std::size_t(i) * d + j] != 0);
        const CodeMatrix c = pack_bits(b);
        std::memcpy(words, c.raw().data(), sizeof(std::uint32_t) * c.raw().size());
    });
}

// unpack_bits (bitcodes.cpp:43-57).
int spotref_unpack_bits(const std::uint32_t* words, std::uint32_t n, std::uint32_t L,
                        std::uint8_t* bits) {
    return guard([&] { copy_bits(unpack_bits(codes_from(words, n, L)), bits); });
}

// nxor_scores_into (bitcodes.cpp:59-76).
int spotref_nxor_scores_into(const std::uint32_t* q, std::uint32_t q_words,
                             const std::uint32_t* words, std::uint32_t n, std::uint32_t L,
                             std::uint32_t n_valid, std::int32_t* out) {
    return guard([&] {
        const CodeMatrix c = codes_from(words, n, L);
        nxor_scores_into({q, q_words}, c, n_valid, out);
    });
}

// top_k_indices<int32_t> (bitcodes.cpp:107-131). out has k entries.
int spotref_top_k_i32(const std::int32_t* scores, std::uint32_t n, std::uint32_t k,
                      std::uint32_t* out) {
    return guard([&] {
        const auto v = top_k_indices<std::int32_t>({scores, n}, k);
        std::memcpy(out, v.data(), sizeof(std::uint32_t) * v.size());
    });
}

int spotref_top_k_f32(const float* scores, std::uint32_t n, std::uint32_t k, std::uint32_t* out) {
    return guard([&] {
        const auto v = top_k_indices<float>({scores, n}, k);
        std::memcpy(out, v.data(), sizeof(std::uint32_t) * v.size());
    });
}

// mlp_forward (hashers.cpp:84-103): x[m][d] -> pre[m][L].
int spotref_mlp_forward(const float* w1, const float* b1, const float* w2, std::uint32_t d,
                        std::uint32_t h, std::uint32_t L, const float* x, std::uint32_t m,
                        float* pre) {
    return guard([&] {
        const Matrix<float> z = mlp_forward(make_mlp(w1, b1, w2, d, h, L), mat(x, m, d));
        std::memcpy(pre, z.data(), sizeof(float) * z.size());
    });
}

// mlp_hash (hashers.cpp:105-108) + pack_bits: x[m][d] -> codes[m][L/32].
int spotref_mlp_hash_packed(const float* w1, const float* b1, const float* w2, std::uint32_t d,
                            std::uint32_t h, std::uint32_t L, const float* x, std::uint32_t m,
                            std::uint32_t* codes) {
    return guard([&] {
        const CodeMatrix c = pack_bits(mlp_hash(make_mlp(w1, b1, w2, d, h, L), mat(x, m, d)));
        std::memcpy(codes, c.raw().data(), sizeof(std::uint32_t) * c.raw().size());
    });
}

// linear_hash (hashers.cpp:75-82) + pack_bits.
int spotref_linear_hash_packed(const float* proj, std::uint32_t d, std::uint32_t L,
                               const float* x, std::uint32_t m, std::uint32_t* codes) {
    return guard([&] {
        LinearHasher lh{mat(proj, d, L)};
        const CodeMatrix c = pack_bits(linear_hash(lh, mat(x, m, d)));
        std::memcpy(codes, c.raw().data(), sizeof(std::uint32_t) * c.raw().size());
    });
}

std::uint32_t spotref_budget_from_rate(double rate, std::uint64_t n, int* status) {
    std::uint32_t k = 0;
    *status = guard([&] { k = budget_from_rate(rate, n); });
    return k;
}

// sparse_attention (attention_eval.cpp:234-264) for q queries against one
// cache. picked is flattened: query r owns picked[off[r] .. off[r+1]).
int spotref_sparse_attention(const float* queries, std::uint32_t q, const float* keys,
                             const float* values, std::uint32_t n, std::uint32_t d, float scale,
                             const std::uint32_t* offsets, const std::uint32_t* picked,
                             const std::uint64_t* picked_off, float* out) {
    return guard([&] {
        AttentionInstance inst;
        inst.queries = mat(queries, q, d);
        inst.keys = mat(keys, n, d);
        inst.values = mat(values, n, d);
        inst.scale = scale;
        inst.causal_offsets.assign(offsets, offsets + q);
        RetrievalResult r;
        r.indices.resize(q);
        for (std::uint32_t i = 0; i < q; ++i)
            r.indices[i].assign(picked + picked_off[i], picked + picked_off[i + 1]);
        const Matrix<float> o = sparse_attention(inst, r);
        std::memcpy(out, o.data(), sizeof(float) * o.size());
    });
}

// full_attention (attention_eval.cpp:101-109).
int spotref_full_attention(const float* queries, std::uint32_t q, const float* keys,
                           const float* values, std::uint32_t n, std::uint32_t d, float scale,
                           const std::uint32_t* offsets, float* out) {
    return guard([&] {
        AttentionInstance inst;
        inst.queries = mat(queries, q, d);
        inst.keys = mat(keys, n, d);
        inst.values = mat(values, n, d);
        inst.scale = scale;
        inst.causal_offsets.assign(offsets, offsets + q);
        const Matrix<float> o = full_attention(inst);
        std::memcpy(out, o.data(), sizeof(float) * o.size());
    });
}

// oracle_topk (attention_eval.cpp:121-135); out[q][k], counts[q].
int spotref_oracle_topk(const float* queries, std::uint32_t q, const float* keys, std::uint32_t n,
                        std::uint32_t d, float scale, const std::uint32_t* offsets, std::uint32_t k,
                        std::uint32_t* out, std::uint32_t* counts) {
    return guard([&] {
        AttentionInstance inst;
        inst.queries = mat(queries, q, d);
        inst.keys = mat(keys, n, d);
        inst.values = mat(keys, n, d);
        inst.scale = scale;
        inst.causal_offsets.assign(offsets, offsets + q);
        const RetrievalResult r = oracle_topk(inst, k);
        for (std::uint32_t i = 0; i < q; ++i) {
            counts[i] = static_cast<std::uint32_t>(r.indices[i].size());
            std::memcpy(out + std::size_t(i) * k, r.indices[i].data(),
                        sizeof(std::uint32_t) * r.indices[i].size());
        }
    });
}

// downproj_topk (attention_eval.cpp:183-206); proj d x r.
int spotref_downproj_topk(const float* queries, std::uint32_t q, const float* keys,
                          std::uint32_t n, std::uint32_t d, const float* proj, std::uint32_t r,
                          const std::uint32_t* offsets, std::uint32_t k, std::uint32_t* out,
                          std::uint32_t* counts) {
    return guard([&] {
        AttentionInstance inst;
        inst.queries = mat(queries, q, d);
        inst.keys = mat(keys, n, d);
        inst.values = mat(keys, n, d);
        inst.scale = 1.0f;
        inst.causal_offsets.assign(offsets, offsets + q);
        DownProjEstimator est;
        est.projection = mat(proj, d, r);
        const RetrievalResult res = downproj_topk(inst, est, k);
        for (std::uint32_t i = 0; i < q; ++i) {
            counts[i] = static_cast<std::uint32_t>(res.indices[i].size());
            std::memcpy(out + std::size_t(i) * k, res.indices[i].data(),
                        sizeof(std::uint32_t) * res.indices[i].size());
        }
    });
}

// evaluate (attention_eval.cpp:285-353) over four methods in this order:
// oracle, mlp (w1 b1 w2), downproj (proj d x r), frozen. stats[4][6] =
// mean_iou, p10, p50, p90, mean_rel_err, max_rel_err; *budget = k.
int spotref_evaluate(const float* queries, std::uint32_t q, const float* keys, const float* values,
                     std::uint32_t n, std::uint32_t d, float scale, const std::uint32_t* offsets,
                     double rate, const float* w1, const float* b1, const float* w2,
                     std::uint32_t h, std::uint32_t L, const float* proj, std::uint32_t r,
                     double* stats, std::uint32_t* budget) {
    return guard([&] {
        AttentionInstance inst;
        inst.queries = mat(queries, q, d);
        inst.keys = mat(keys, n, d);
        inst.values = mat(values, n, d);
        inst.scale = scale;
        inst.causal_offsets.assign(offsets, offsets + q);
        const AnyHasher mlp = make_mlp(w1, b1, w2, d, h, L);
        DownProjEstimator est;
        est.projection = mat(proj, d, r);
        const AnyHasher dp = est;
        std::vector<EvalMethodSpec> ms(4);
        ms[0].name = "oracle";
        ms[0].kind = RetrievalMethod::oracle;
        ms[1].name = "mlp";
        ms[1].kind = RetrievalMethod::mlp;
        ms[1].hasher = &mlp;
        ms[2].name = "downproj";
        ms[2].kind = RetrievalMethod::downproj;
        ms[2].hasher = &dp;
        ms[3].name = "full";
        ms[3].kind = RetrievalMethod::oracle;
        ms[3].frozen = true;
        const EvalReport rep = evaluate(inst, ms, rate);
        *budget = rep.budget;
        for (int i = 0; i < 4; ++i) {
            const MethodReport& m = rep.methods[i];
            const double v[6] = {m.mean_iou, m.p10_iou, m.p50_iou, m.p90_iou, m.mean_rel_err,
                                 m.max_rel_err};
            for (int j = 0; j < 6; ++j) stats[i * 6 + j] = v[j];
        }
    });
}

// iou (attention_eval.cpp:216-232) of two ascending index lists.
double spotref_iou(const std::uint32_t* a, std::uint32_t na, const std::uint32_t* b,
                   std::uint32_t nb) {
    return iou({a, na}, {b, nb});
}

// hash_topk (attention_eval.cpp:137-181) with an MLP hasher; out[q][k]
// (each row holds min(k, offset) indices; the rest untouched).
int spotref_hash_topk_mlp(const float* w1, const float* b1, const float* w2, std::uint32_t h,
                          std::uint32_t L, const float* queries, std::uint32_t q,
                          const float* keys, const float* values, std::uint32_t n,
                          std::uint32_t d, float scale, const std::uint32_t* offsets,
                          std::uint32_t k, std::uint32_t* out, std::uint32_t* counts) {
    return guard([&] {
        AttentionInstance inst;
        inst.queries = mat(queries, q, d);
        inst.keys = mat(keys, n, d);
        inst.values = mat(values, n, d);
        inst.scale = scale;
        inst.causal_offsets.assign(offsets, offsets + q);
        const AnyHasher hh = make_mlp(w1, b1, w2, d, h, L);
        const RetrievalResult r = hash_topk(inst, hh, k);
        for (std::uint32_t i = 0; i < q; ++i) {
            counts[i] = static_cast<std::uint32_t>(r.indices[i].size());
            std::memcpy(out + std::size_t(i) * k, r.indices[i].data(),
                        sizeof(std::uint32_t) * r.indices[i].size());
        }
    });
}

// The reference's decode-time retrieval for P independent (batch, head)
// problems, the CPU baseline arm of bench.py. spotref_index_create builds one
// reference CodeMatrix per problem ONCE (the resident code cache, outside any
// timed region); spotref_retrieve_batch then runs, per problem,
// nxor_scores_into + top_k_indices exactly as hash_topk composes them
// (attention_eval.cpp:172-179), problems spread over OpenMP threads
// (result-independent partitioning).
struct SpotrefIndex {
    std::vector<CodeMatrix> per_problem;
    std::uint32_t L = 0;
};

int spotref_index_create(const std::uint32_t* codes, std::uint32_t P, std::uint64_t cap,
                         std::uint32_t L, const std::uint32_t* n_rows, void** out) {
    return guard([&] {
        auto* idx = new SpotrefIndex;
        idx->L = L;
        const std::uint32_t W = L / 32;
        idx->per_problem.reserve(P);
        for (std::uint32_t p = 0; p < P; ++p) {
            CodeMatrix c(n_rows[p], L);
            std::memcpy(c.raw().data(), codes + std::size_t(p) * cap * W,
                        sizeof(std::uint32_t) * std::size_t(n_rows[p]) * W);
            idx->per_problem.push_back(std::move(c));
        }
        *out = idx;
    });
}

void spotref_index_destroy(void* h) { delete static_cast<SpotrefIndex*>(h); }

int spotref_retrieve_batch(void* handle, const std::uint32_t* qcodes,
                           const std::uint32_t* n_valid, std::uint32_t k, std::uint32_t* out,
                           int threads) {
    return guard([&] {
        auto* idx = static_cast<SpotrefIndex*>(handle);
        const std::uint32_t P = static_cast<std::uint32_t>(idx->per_problem.size());
        const std::uint32_t W = idx->L / 32;
        int status = 0;
        std::string err;
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
        {
            std::vector<std::int32_t> scores;
#pragma omp for schedule(dynamic, 1)
            for (std::uint32_t p = 0; p < P; ++p) {
                try {
                    const CodeMatrix& c = idx->per_problem[p];
                    const std::uint32_t n = n_valid[p];
                    scores.resize(c.rows());
                    nxor_scores_into({qcodes + std::size_t(p) * W, W}, c, n, scores.data());
                    const std::uint32_t kk = std::min<std::uint32_t>(k, n);
                    const auto v = top_k_indices<std::int32_t>({scores.data(), n}, kk);
                    std::memcpy(out + std::size_t(p) * k, v.data(),
                                sizeof(std::uint32_t) * v.size());
                } catch (const std::exception& e) {
#pragma omp critical
                    {
                        status = 1;
                        err = e.what();
                    }
                }
            }
        }
        if (status) throw DimensionError(err);
    });
}

// ------------------------------------------------------------ trainer (§8 f4)
// train_hasher (trainer.cpp:634-645) on an MLP hasher. Sequences are
// concatenated: sequence s has seq_len[s] query rows and as many key rows.
// dcfg = {max_lr, min_lr, adam_beta1, adam_beta2, adam_eps, weight_decay,
//         grad_clip, soft_gamma, holdout_budget_rate, beta, alpha, maskout}
// ucfg = {num_iters, warmup_iters, batch, seed, holdout_queries}
// opt  = {max_top, max_oth, query_subsample} (-1: unset)
// rec  = num_iters x {loss, violation_rate, lr}
// kind: 1 MLP (w1 d x h, b1, w2 h x L), 0 linear / 2 downproj (w1 = projection d x L).
int spotref_train(int kind, float* w1, float* b1, float* w2, std::uint32_t d, std::uint32_t h,
                  std::uint32_t L, float gamma, std::uint32_t n_seq, const float* queries,
                  const float* keys, const std::uint32_t* seq_len, const double* dcfg,
                  const std::uint64_t* ucfg, const std::int64_t* opt, int loss_kind,
                  double* rec, double* holdout_iou, std::uint32_t* skipped) {
    return guard([&] {
        AnyHasher any;
        if (kind == 1) {
            MlpHasher m;
            m.w1 = mat(w1, d, h);
            m.b1.assign(b1, b1 + h);
            m.w2 = mat(w2, h, L);
            m.gamma = gamma;
            any = m;
        } else if (kind == 0) {
            any = LinearHasher{mat(w1, d, L)};
        } else {
            any = DownProjEstimator{mat(w1, d, L)};
        }
        TrainDataset data;
        std::size_t off = 0;
        for (std::uint32_t s = 0; s < n_seq; ++s) {
            data.sequences.push_back(QkSequence{mat(queries + off * d, seq_len[s], d),
                                                mat(keys + off * d, seq_len[s], d)});
            off += seq_len[s];
        }
        TrainConfig cfg;
        cfg.max_lr = dcfg[0];
        cfg.min_lr = dcfg[1];
        cfg.adam_beta1 = dcfg[2];
        cfg.adam_beta2 = dcfg[3];
        cfg.adam_eps = dcfg[4];
        cfg.weight_decay = dcfg[5];
        cfg.grad_clip = dcfg[6];
        cfg.soft_gamma = dcfg[7];
        cfg.holdout_budget_rate = dcfg[8];
        cfg.num_iters = static_cast<std::uint32_t>(ucfg[0]);
        cfg.warmup_iters = static_cast<std::uint32_t>(ucfg[1]);
        cfg.batch = static_cast<std::uint32_t>(ucfg[2]);
        cfg.seed = ucfg[3];
        cfg.holdout_queries = static_cast<std::uint32_t>(ucfg[4]);
        RankingLossConfig lc;
        lc.beta = dcfg[9];
        lc.alpha = dcfg[10];
        lc.maskout = dcfg[11];
        if (opt[0] >= 0) lc.max_top = static_cast<std::uint32_t>(opt[0]);
        if (opt[1] >= 0) lc.max_oth = static_cast<std::uint32_t>(opt[1]);
        if (opt[2] >= 0) lc.query_subsample = static_cast<std::uint32_t>(opt[2]);
        const TrainReport r = train_hasher(
            any, data, lc, cfg, loss_kind == 1 ? TrainLoss::reconstruction : TrainLoss::ranking);
        if (kind == 1) {
            const MlpHasher& out = std::get<MlpHasher>(any);
            std::memcpy(w1, out.w1.data(), sizeof(float) * d * h);
            std::memcpy(b1, out.b1.data(), sizeof(float) * h);
            std::memcpy(w2, out.w2.data(), sizeof(float) * h * L);
        } else if (kind == 0) {
            std::memcpy(w1, std::get<LinearHasher>(any).projection.data(), sizeof(float) * d * L);
        } else {
            std::memcpy(w1, std::get<DownProjEstimator>(any).projection.data(), sizeof(float) * d * L);
        }
        for (std::size_t i = 0; i < r.records.size(); ++i) {
            rec[3 * i] = r.records[i].loss;
            rec[3 * i + 1] = r.records[i].violation_rate;
            rec[3 * i + 2] = r.records[i].lr;
        }
        *holdout_iou = r.final_holdout_iou;
        *skipped = r.skipped_steps;
    });
}

// partition_topk (ranking_loss.cpp:80-145) over an identity order (row i of
// the order = 0..n-1), so the returned key indices ARE the sampled positions:
// the host sampler of the GPU trainer is checked against this.
int spotref_partition_identity(std::uint32_t q, std::uint32_t n, const std::uint32_t* offsets,
                               const double* bam, const std::int64_t* opt, std::uint64_t seed,
                               std::uint32_t* rows_out, std::uint32_t* top_out,
                               std::uint32_t* oth_out, std::uint32_t* counts,
                               std::uint64_t* valid_pairs) {
    return guard([&] {
        TopkOrder o;
        o.n_keys = n;
        o.n_queries = q;
        o.causal_offsets.assign(offsets, offsets + q);
        o.order.resize(std::size_t(q) * n);
        for (std::size_t r = 0; r < q; ++r)
            for (std::uint32_t j = 0; j < n; ++j) o.order[r * n + j] = j;
        RankingLossConfig lc;
        lc.beta = bam[0];
        lc.alpha = bam[1];
        lc.maskout = bam[2];
        if (opt[0] >= 0) lc.max_top = static_cast<std::uint32_t>(opt[0]);
        if (opt[1] >= 0) lc.max_oth = static_cast<std::uint32_t>(opt[1]);
        if (opt[2] >= 0) lc.query_subsample = static_cast<std::uint32_t>(opt[2]);
        const PairPartition p = partition_topk(o, lc, seed);
        counts[0] = static_cast<std::uint32_t>(p.query_rows.size());
        counts[1] = p.top_count;
        counts[2] = p.oth_count;
        counts[3] = p.k_full;
        std::copy(p.query_rows.begin(), p.query_rows.end(), rows_out);
        for (std::uint32_t i = 0; i < p.top_count; ++i) top_out[i] = p.top_indices[i];
        for (std::uint32_t j = 0; j < p.oth_count; ++j) oth_out[j] = p.oth_indices[j] - p.k_full;
        *valid_pairs = p.valid_pairs;
    });
}

double spotref_lr_at(std::uint32_t iter, std::uint32_t num_iters, std::uint32_t warmup,
                     double max_lr, double min_lr) {
    TrainConfig cfg;
    cfg.num_iters = num_iters;
    cfg.warmup_iters = warmup;
    cfg.max_lr = max_lr;
    cfg.min_lr = min_lr;
    return lr_at(iter, cfg);
}

}  // extern "C"
