// C++ parity tests of the drop-in spotlight:: API (libspotlight_b200.so, GPU)
// written like the reference's own doctest suite
// (proj/tests/test_bitcodes.cpp, test_hashers.cpp, test_attention_eval.cpp),
// plus bit-exact differential checks against the unmodified reference
// (oracle/_ref/libspotref.so via its extern "C" shim) when it was built.
// Run by tests/test_gpu_dropin.py; exit code = number of failed checks.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numeric>
#include <random>
#include <string>
#include <unistd.h>
#include <thread>
#include <vector>

#include "spotlight/attention_eval.hpp"
#include "spotlight/bitcodes.hpp"
#include "spotlight/errors.hpp"
#include "spotlight/hashers.hpp"
#include "spotlight/synthkv.hpp"
#include "spotlight/trainer.hpp"

using namespace spotlight;

// ------------------------------------------------------------ mini harness
static int g_checks = 0, g_failed = 0;
static const char* g_case = "";
#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_failed;                                                               \
            std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond); \
        }                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, Exc)                                 \
    do {                                                           \
        bool thrown_ = false;                                      \
        try {                                                      \
            (void)(expr);                                          \
        } catch (const Exc&) {                                     \
            thrown_ = true;                                        \
        } catch (...) {                                            \
        }                                                          \
        CHECK(thrown_ && #Exc);                                    \
    } while (0)
#define CHECK_THROWS_WITH(expr, Exc, needle)                                  \
    do {                                                                      \
        bool ok_ = false;                                                     \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (const Exc& e) {                                              \
            ok_ = std::string(e.what()).find(needle) != std::string::npos;    \
        } catch (...) {                                                       \
        }                                                                     \
        CHECK(ok_ && "exception message");                                    \
    } while (0)

static std::vector<std::pair<const char*, std::function<void()>>>& registry() {
    static std::vector<std::pair<const char*, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name)                                   \
    static void CAT(tc_, __LINE__)();                     \
    static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
    static void CAT(tc_, __LINE__)()

// ------------------------------------------------------------ helpers
static BitMatrix random_bits(std::size_t n, std::size_t d, std::mt19937_64& eng) {
    BitMatrix b(n, d);
    std::bernoulli_distribution coin(0.5);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < d; ++j) b.set(i, j, coin(eng));
    return b;
}
static Matrix<float> random_matrix(std::size_t r, std::size_t c, std::mt19937_64& eng, double s = 1.0) {
    std::normal_distribution<double> g(0.0, s);
    Matrix<float> m(r, c);
    for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = static_cast<float>(g(eng));
    return m;
}
static std::vector<std::uint32_t> full_sort_topk(const std::vector<std::int32_t>& s, std::uint32_t k) {
    std::vector<std::uint32_t> idx(s.size());
    std::iota(idx.begin(), idx.end(), 0u);
    std::sort(idx.begin(), idx.end(), [&](std::uint32_t a, std::uint32_t b) {
        return s[a] != s[b] ? s[a] > s[b] : a < b;
    });
    idx.resize(k);
    std::sort(idx.begin(), idx.end());
    return idx;
}
static AttentionInstance random_instance(std::size_t q, std::size_t n, std::size_t d,
                                         std::mt19937_64& eng, bool causal) {
    AttentionInstance inst;
    inst.queries = random_matrix(q, d, eng);
    inst.keys = random_matrix(n, d, eng);
    inst.values = random_matrix(n, d, eng);
    inst.scale = 1.0f / std::sqrt(static_cast<float>(d));
    inst.causal_offsets.resize(q);
    for (std::size_t i = 0; i < q; ++i)
        inst.causal_offsets[i] = causal ? static_cast<std::uint32_t>(std::min(i + 1, n))
                                        : static_cast<std::uint32_t>(n);
    return inst;
}

// ------------------------------------------------------------ bitcodes
TEST_CASE("pack_bits single-word examples") {
    BitMatrix one(1, 32);
    one.set(0, 0, true);
    CHECK(pack_bits(one).row(0)[0] == 0x80000000u);
    CHECK(pack_bits(BitMatrix(1, 32)).row(0)[0] == 0u);
    BitMatrix wide(1, 64);
    wide.set(0, 1, true);
    const CodeMatrix c = pack_bits(wide);
    CHECK(c.row(0)[0] == 0u);
    CHECK(c.row(0)[1] == 0x80000000u);
}

TEST_CASE("pack_bits rejects widths that are not multiples of 32") {
    CHECK_THROWS_AS(pack_bits(BitMatrix(1, 33)), DimensionError);
    CHECK_THROWS_AS(pack_bits(BitMatrix(1, 0)), DimensionError);
}

TEST_CASE("pack_bits layout oracle and unpack round trip") {
    std::mt19937_64 eng(7);
    for (int it = 0; it < 60; ++it) {
        const std::size_t n = 1 + eng() % 8, d = 32 * (1 + eng() % 8);
        const BitMatrix bits = random_bits(n, d, eng);
        const CodeMatrix got = pack_bits(bits);
        CodeMatrix want(static_cast<std::uint32_t>(n), static_cast<std::uint32_t>(d));
        const std::size_t cw = d / 32;
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t j = 0; j < d; ++j)
                if (bits.get(i, j)) want.row(static_cast<std::uint32_t>(i))[j % cw] |= 1u << (31 - j / cw);
        CHECK(got == want);
        CHECK(unpack_bits(got) == bits);
    }
}

TEST_CASE("nxor_scores counts agreeing bits") {
    std::mt19937_64 eng(13);
    const BitMatrix bits = random_bits(8, 128, eng);
    const CodeMatrix codes = pack_bits(bits);
    CHECK(nxor_scores(codes.code(3), codes)[3] == 128);
    BitMatrix flipped = bits;
    for (std::size_t j = 0; j < 128; ++j) flipped.set(0, j, !bits.get(0, j));
    CHECK(nxor_scores(pack_bits(flipped).code(0), codes)[0] == 0);
    const CodeMatrix other(4, 64);
    CHECK_THROWS_AS(nxor_scores(other.code(0), codes), DimensionError);
}

TEST_CASE("affine identity 2m - L == signed dot product") {
    std::mt19937_64 eng(17);
    for (int it = 0; it < 40; ++it) {
        const std::size_t d = 32 * (1 + eng() % 8);
        const BitMatrix bits = random_bits(6, d, eng);
        const ScoreVector s = nxor_scores(pack_bits(bits).code(0), pack_bits(bits));
        for (std::size_t r = 0; r < 6; ++r) {
            int dot = 0;
            for (std::size_t j = 0; j < d; ++j) dot += (bits.get(0, j) ? 1 : -1) * (bits.get(r, j) ? 1 : -1);
            CHECK(2 * s[r] - static_cast<int>(d) == dot);
        }
    }
}

TEST_CASE("top_k_indices examples, tie rule and full-sort oracle") {
    CHECK(top_k_indices(ScoreVector{3, 1, 2}, 1) == std::vector<std::uint32_t>{0});
    CHECK(top_k_indices(ScoreVector{2, 2, 1}, 1) == std::vector<std::uint32_t>{0});
    CHECK((top_k_indices(ScoreVector{5, 9, 1, 7}, 4) == std::vector<std::uint32_t>{0, 1, 2, 3}));
    CHECK_THROWS_WITH(top_k_indices(ScoreVector{3, 1, 2}, 0), DimensionError, "k=0 out of range for n=3");
    CHECK_THROWS_AS(top_k_indices(ScoreVector{3, 1, 2}, 4), DimensionError);
    std::mt19937_64 eng(23);
    for (int it = 0; it < 100; ++it) {
        const std::size_t n = 1 + eng() % 257;
        std::uniform_int_distribution<std::int32_t> sc(0, 12);
        ScoreVector s(n);
        for (auto& v : s) v = sc(eng);
        const std::uint32_t k = 1 + eng() % n;
        CHECK(top_k_indices(s, k) == full_sort_topk(s, k));
    }
    std::uniform_int_distribution<std::int32_t> sc(0, 128);
    ScoreVector s(10000);
    for (auto& v : s) v = sc(eng);
    for (std::uint32_t k : {1u, 17u, 200u, 9999u, 10000u}) CHECK(top_k_indices(s, k) == full_sort_topk(s, k));
    const std::vector<float> f{0.5f, -0.0f, 0.0f, 0.5f, -1.0f};
    CHECK((top_k_indices<float>(std::span<const float>(f), 3) == std::vector<std::uint32_t>{0, 1, 3}));
}

TEST_CASE("SPLC round trip and validation") {
    std::mt19937_64 eng(29);
    const CodeMatrix codes = pack_bits(random_bits(17, 96, eng));
    const std::string path = "test_dropin_codes.splc";
    write_code_index(path, codes);
    CHECK(read_code_index(path) == codes);
    {
        FILE* f = std::fopen(path.c_str(), "r+b");
        std::fputc('X', f);
        std::fclose(f);
        CHECK_THROWS_WITH(read_code_index(path), FormatError, "offset 0");
    }
    write_code_index(path, codes);
    {
        FILE* f = std::fopen(path.c_str(), "r+b");
        CHECK(ftruncate(fileno(f), 24) == 0);
        std::fclose(f);
        CHECK_THROWS_AS(read_code_index(path), FormatError);
    }
    std::remove(path.c_str());
}

// ------------------------------------------------------------ hashers
TEST_CASE("mlp_hash sign behaviour") {
    std::mt19937_64 eng(37);
    MlpHasher zero;
    zero.w1 = Matrix<float>(8, 8);
    zero.b1.assign(8, 0.0f);
    zero.w2 = Matrix<float>(8, 32);
    const BitMatrix ones = mlp_hash(zero, random_matrix(2, 8, eng));
    bool all = true;
    for (std::size_t i = 0; i < ones.rows(); ++i)
        for (std::size_t j = 0; j < ones.cols(); ++j) all = all && ones.get(i, j);
    CHECK(all);
    const MlpHasher h = mlp_gaussian_init(16, 16, 32, 64.0f, 5);
    const Matrix<float> x = random_matrix(7, 16, eng, 3.0);
    const Matrix<float> pre = mlp_forward(h, x);
    const BitMatrix bits = mlp_hash(h, x);
    bool same = true;
    for (std::size_t i = 0; i < pre.rows(); ++i)
        for (std::size_t j = 0; j < pre.cols(); ++j) same = same && (bits.get(i, j) == (pre(i, j) >= 0.0f));
    CHECK(same);
    MlpHasher scaled = mlp_gaussian_init(16, 16, 32, 64.0f, 9);
    const BitMatrix before = mlp_hash(scaled, x);
    for (std::size_t i = 0; i < scaled.w2.size(); ++i) scaled.w2.data()[i] *= 7.5f;
    CHECK(mlp_hash(scaled, x) == before);
}

TEST_CASE("non-finite input and weights are rejected") {
    MlpHasher h = mlp_gaussian_init(4, 4, 32, 64.0f, 3);
    Matrix<float> x(1, 4);
    x(0, 2) = std::nanf("");
    CHECK_THROWS_WITH(mlp_forward(h, x), NumericError, "mlp input contains non-finite values");
    h.w2(0, 0) = INFINITY;
    CHECK_THROWS_AS(mlp_forward(h, Matrix<float>(1, 4)), NumericError);
}

TEST_CASE("hamming score equals (signed dot + L) / 2 on MLP codes") {
    std::mt19937_64 eng(47);
    const MlpHasher h = mlp_gaussian_init(16, 16, 32, 64.0f, 13);
    const BitMatrix bits = mlp_hash(h, random_matrix(10, 16, eng, 2.0));
    const ScoreVector s = nxor_scores(pack_bits(bits).code(0), pack_bits(bits));
    for (std::size_t r = 0; r < bits.rows(); ++r) {
        int dot = 0;
        for (std::size_t j = 0; j < bits.cols(); ++j) dot += (bits.get(0, j) ? 1 : -1) * (bits.get(r, j) ? 1 : -1);
        CHECK(s[r] == (dot + 32) / 2);
    }
}

TEST_CASE("hashing is deterministic across repeated calls") {
    std::mt19937_64 eng(59);
    const MlpHasher h = mlp_gaussian_init(32, 32, 32, 64.0f, 17);
    const Matrix<float> x = random_matrix(64, 32, eng, 2.0);
    const BitMatrix first = mlp_hash(h, x);
    for (int i = 0; i < 3; ++i) CHECK(mlp_hash(h, x) == first);
}

TEST_CASE("SPLH checkpoint round trips") {
    const std::string path = "test_dropin_hasher.splh";
    const MlpHasher h = mlp_gaussian_init(8, 12, 32, 48.0f, 23);
    write_hasher(path, h);
    const AnyHasher back = read_hasher(path);
    CHECK(std::holds_alternative<MlpHasher>(back));
    const auto& m = std::get<MlpHasher>(back);
    CHECK(m.w1 == h.w1);
    CHECK(m.b1 == h.b1);
    CHECK(m.w2 == h.w2);
    CHECK(m.gamma == h.gamma);
    CHECK(std::string(hasher_kind_name(back)) == "mlp");
    std::remove(path.c_str());
}

// ------------------------------------------------------------ attention_eval
TEST_CASE("budget_from_rate applies floor and clamp") {
    CHECK(budget_from_rate(0.02, 2048) == 40);
    CHECK(budget_from_rate(0.02, 500) == 20);
    CHECK(budget_from_rate(1.0, 8) == 8);
    CHECK_THROWS_AS(budget_from_rate(0.0, 10), DimensionError);
}

TEST_CASE("sparse_attention over the full set reproduces full attention") {
    std::mt19937_64 eng(11);
    const AttentionInstance inst = random_instance(6, 32, 16, eng, true);
    RetrievalResult all;
    all.indices.resize(6);
    for (std::size_t r = 0; r < 6; ++r) {
        all.indices[r].resize(inst.causal_offsets[r]);
        std::iota(all.indices[r].begin(), all.indices[r].end(), 0u);
    }
    const Matrix<float> sp = sparse_attention(inst, all), fu = full_attention(inst);
    for (std::size_t r = 0; r < 6; ++r) {
        double d2 = 0, n2 = 0;
        for (std::size_t p = 0; p < 16; ++p) {
            d2 += (sp(r, p) - fu(r, p)) * (sp(r, p) - fu(r, p));
            n2 += fu(r, p) * fu(r, p);
        }
        CHECK(std::sqrt(d2) <= 1e-6 * std::sqrt(n2));
    }
}

TEST_CASE("own token is always attended; rejections") {
    std::mt19937_64 eng(11);
    const AttentionInstance inst = random_instance(4, 4, 8, eng, true);
    RetrievalResult own;
    own.indices = {{0}, {1}, {2}, {3}};
    const Matrix<float> o = sparse_attention(inst, own);
    for (std::size_t p = 0; p < 8; ++p) CHECK(std::fabs(o(0, p) - inst.values(0, p)) < 1e-6f);
    RetrievalResult empty;
    empty.indices = {{0}, {}, {0}, {0}};
    CHECK_THROWS_AS(sparse_attention(inst, empty), DimensionError);
    RetrievalResult out_of_range;
    out_of_range.indices = {{3}, {0}, {0}, {0}};
    CHECK_THROWS_AS(sparse_attention(inst, out_of_range), DimensionError);
}

TEST_CASE("hash_topk: duplicated keys keep the lower index; collapsed hasher -> first k") {
    std::mt19937_64 eng(13);
    AttentionInstance inst = random_instance(2, 8, 32, eng, false);
    for (std::size_t p = 0; p < 32; ++p) inst.keys(4, p) = inst.keys(1, p);
    LinearHasher lin{random_matrix(32, 32, eng)};
    const RetrievalResult a = hash_topk(inst, lin, 3), b = hash_topk(inst, lin, 3);
    CHECK(a.indices == b.indices);
    for (const auto& idx : a.indices)
        if (std::find(idx.begin(), idx.end(), 4u) != idx.end())
            CHECK(std::find(idx.begin(), idx.end(), 1u) != idx.end());
    const AttentionInstance big = random_instance(64, 512, 32, eng, false);
    MlpHasher collapsed;
    collapsed.w1 = Matrix<float>(32, 8);
    collapsed.b1.assign(8, 0.0f);
    collapsed.w2 = Matrix<float>(8, 32);
    const RetrievalResult res = hash_topk(big, collapsed, 16);
    std::vector<std::uint32_t> first(16);
    std::iota(first.begin(), first.end(), 0u);
    for (const auto& idx : res.indices) CHECK(idx == first);
    CHECK_THROWS_AS(hash_topk(big, DownProjEstimator{Matrix<float>(32, 4)}, 16), DimensionError);
    CHECK_THROWS_AS(hash_topk(big, collapsed, 0), DimensionError);
}

// ------------------------------------------------------------ vs the reference
struct Ref {
    void* h = nullptr;
    int (*mlp_forward)(const float*, const float*, const float*, std::uint32_t, std::uint32_t,
                       std::uint32_t, const float*, std::uint32_t, float*) = nullptr;
    int (*hash_topk)(const float*, const float*, const float*, std::uint32_t, std::uint32_t,
                     const float*, std::uint32_t, const float*, const float*, std::uint32_t,
                     std::uint32_t, float, const std::uint32_t*, std::uint32_t, std::uint32_t*,
                     std::uint32_t*) = nullptr;
    int (*sparse)(const float*, std::uint32_t, const float*, const float*, std::uint32_t,
                  std::uint32_t, float, const std::uint32_t*, const std::uint32_t*,
                  const std::uint64_t*, float*) = nullptr;
    int (*oracle)(const float*, std::uint32_t, const float*, std::uint32_t, std::uint32_t, float,
                  const std::uint32_t*, std::uint32_t, std::uint32_t*, std::uint32_t*) = nullptr;
    int (*downproj)(const float*, std::uint32_t, const float*, std::uint32_t, std::uint32_t,
                    const float*, std::uint32_t, const std::uint32_t*, std::uint32_t,
                    std::uint32_t*, std::uint32_t*) = nullptr;
    int (*train)(int, float*, float*, float*, std::uint32_t, std::uint32_t, std::uint32_t, float,
                 std::uint32_t, const float*, const float*, const std::uint32_t*, const double*,
                 const std::uint64_t*, const std::int64_t*, int, double*, double*,
                 std::uint32_t*) = nullptr;
    int (*evaluate)(const float*, std::uint32_t, const float*, const float*, std::uint32_t,
                    std::uint32_t, float, const std::uint32_t*, double, const float*,
                    const float*, const float*, std::uint32_t, std::uint32_t, const float*,
                    std::uint32_t, double*, std::uint32_t*) = nullptr;
    Ref() {
        const char* p = std::getenv("SPOTREF_SO");
        h = dlopen(p ? p : "oracle/_ref/libspotref.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        mlp_forward = reinterpret_cast<decltype(mlp_forward)>(dlsym(h, "spotref_mlp_forward"));
        hash_topk = reinterpret_cast<decltype(hash_topk)>(dlsym(h, "spotref_hash_topk_mlp"));
        sparse = reinterpret_cast<decltype(sparse)>(dlsym(h, "spotref_sparse_attention"));
        oracle = reinterpret_cast<decltype(oracle)>(dlsym(h, "spotref_oracle_topk"));
        downproj = reinterpret_cast<decltype(downproj)>(dlsym(h, "spotref_downproj_topk"));
        evaluate = reinterpret_cast<decltype(evaluate)>(dlsym(h, "spotref_evaluate"));
        train = reinterpret_cast<decltype(train)>(dlsym(h, "spotref_train"));
    }
};

// softmax weights of one query over its causal range (f64; monotone in the logits)
static std::vector<double> soft_weights(const AttentionInstance& inst, std::size_t row) {
    const std::size_t d = inst.keys.cols(), n = inst.causal_offsets[row];
    std::vector<double> lg(n);
    double mx = -1e300;
    for (std::size_t j = 0; j < n; ++j) {
        double a = 0.0;
        for (std::size_t p = 0; p < d; ++p) a += double(inst.queries(row, p)) * inst.keys(j, p);
        lg[j] = a * inst.scale;
        mx = std::max(mx, lg[j]);
    }
    double s = 0.0;
    for (double& v : lg) s += (v = std::exp(v - mx));
    for (double& v : lg) v /= s;
    return lg;
}

TEST_CASE("oracle_topk agrees with an exhaustive sort; one dropped key obeys the leak-mass relation") {
    std::mt19937_64 eng(4242);
    for (int iter = 0; iter < 30; ++iter) {
        const std::size_t n = 5 + eng() % 60;
        const AttentionInstance inst = random_instance(4, n, 8, eng, iter % 2 == 0);
        const std::uint32_t k = 1 + eng() % 5;
        const RetrievalResult res = oracle_topk(inst, k);
        for (std::size_t row = 0; row < 4; ++row) {
            const auto w = soft_weights(inst, row);
            std::vector<std::uint32_t> order(w.size());
            std::iota(order.begin(), order.end(), 0u);
            std::sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
                return w[a] != w[b] ? w[a] > w[b] : a < b;
            });
            order.resize(std::min<std::size_t>(k, w.size()));
            std::sort(order.begin(), order.end());
            CHECK(res.indices[row] == order);
        }
    }
    for (int iter = 0; iter < 30; ++iter) {
        const std::size_t n = 8 + eng() % 24;
        const AttentionInstance inst = random_instance(1, n, 8, eng, false);
        const RetrievalResult res = oracle_topk(inst, static_cast<std::uint32_t>(n - 1));
        const auto w = soft_weights(inst, 0);
        std::vector<char> kept(n, 0);
        for (auto i : res.indices[0]) kept[i] = 1;
        std::size_t drop = 0;
        for (std::size_t j = 0; j < n; ++j)
            if (!kept[j]) drop = j;
        if (drop == n - 1) continue;  // the own row is always attended: nothing dropped
        const Matrix<float> sp = sparse_attention(inst, res), full = full_attention(inst);
        double diff2 = 0.0, gap2 = 0.0;
        for (std::size_t p = 0; p < 8; ++p) {
            const double dl = double(sp(0, p)) - full(0, p), g = double(inst.values(drop, p)) - sp(0, p);
            diff2 += dl * dl;
            gap2 += g * g;
        }
        // one dropped key: full - sparse == w_drop * (v_drop - sparse)
        CHECK(std::fabs(std::sqrt(diff2) - w[drop] * std::sqrt(gap2)) <= 1e-3 * w[drop] * std::sqrt(gap2) + 1e-6);
    }
}

TEST_CASE("concurrent callers: each host thread gets its own context (SPEC.md:88-89)") {
    std::mt19937_64 eng(555);
    const std::uint32_t n = 400, d = 64;
    std::vector<AttentionInstance> insts;
    for (int t = 0; t < 4; ++t)
        insts.push_back(make_causal_instance(random_matrix(n, d, eng), random_matrix(n, d, eng),
                                             random_matrix(n, d, eng)));
    const MlpHasher h = mlp_gaussian_init(d, d, 128, 64.0f, 8);
    std::vector<RetrievalResult> seq(4), par(4);
    std::vector<Matrix<float>> seq_out, par_out(4);
    for (int t = 0; t < 4; ++t) {
        seq[t] = hash_topk(insts[t], h, 24);
        seq_out.push_back(sparse_attention(insts[t], seq[t]));
    }
    std::vector<std::thread> th;
    for (int t = 0; t < 4; ++t)
        th.emplace_back([&, t] {
            for (int rep = 0; rep < 3; ++rep) {
                par[t] = hash_topk(insts[t], h, 24);
                par_out[t] = sparse_attention(insts[t], par[t]);
            }
        });
    for (auto& x : th) x.join();
    for (int t = 0; t < 4; ++t) {
        CHECK(par[t].indices == seq[t].indices);
        CHECK(std::memcmp(par_out[t].data(), seq_out[t].data(), seq_out[t].size() * 4) == 0);
    }
}

TEST_CASE("downproj_topk and evaluate: exact retrieval, report statistics, formatting") {
    std::mt19937_64 eng(91);
    const std::uint32_t n = 700, d = 64, r = 16, L = 128;
    AttentionInstance inst = make_causal_instance(random_matrix(n, d, eng), random_matrix(n, d, eng),
                                                  random_matrix(n, d, eng));
    DownProjEstimator est{random_matrix(d, r, eng)};
    const RetrievalResult dp = downproj_topk(inst, est, 40);
    CHECK(dp.method == RetrievalMethod::downproj);
    CHECK(dp.indices[n - 1].size() == 40);
    CHECK_THROWS_AS(downproj_topk(inst, est, 0), DimensionError);
    CHECK_THROWS_AS(downproj_topk(inst, DownProjEstimator{random_matrix(d + 1, r, eng)}, 4),
                    DimensionError);
    const MlpHasher mh = mlp_gaussian_init(d, d, L, 64.0f, 12);
    const AnyHasher mlp = mh, dph = est;
    std::vector<EvalMethodSpec> ms(4);
    ms[0].name = "oracle";
    ms[1].name = "mlp";
    ms[1].kind = RetrievalMethod::mlp;
    ms[1].hasher = &mlp;
    ms[2].name = "downproj";
    ms[2].kind = RetrievalMethod::downproj;
    ms[2].hasher = &dph;
    ms[3].name = "full";
    ms[3].frozen = true;
    const EvalReport rep = evaluate(inst, ms, 0.05);
    CHECK(rep.budget == budget_from_rate(0.05, n));
    CHECK(rep.methods.size() == 4);
    CHECK(rep.methods[0].mean_iou == 1.0);            // the oracle against itself
    CHECK(rep.methods[3].max_rel_err < 1e-5);         // every row attended == full attention
    const std::vector<std::string> hdr = {"provenance line"};
    const std::string txt = format_eval_report(rep, hdr);
    CHECK(txt.rfind("# provenance line\nbudget ", 0) == 0);
    CHECK(txt.find("method mlp kind=mlp budget=") != std::string::npos);
    CHECK(eval_report_csv(rep).rfind("query,oracle,mlp,downproj,full\n0,", 0) == 0);
    static Ref ref;
    if (!ref.h || !ref.downproj || !ref.evaluate) return;
    std::vector<std::uint32_t> ridx(static_cast<std::size_t>(n) * 40), rcnt(n);
    CHECK(ref.downproj(inst.queries.data(), n, inst.keys.data(), n, d, est.projection.data(), r,
                       inst.causal_offsets.data(), 40, ridx.data(), rcnt.data()) == 0);
    bool same = true;
    for (std::uint32_t q = 0; q < n; ++q)
        same = same && dp.indices[q] == std::vector<std::uint32_t>(ridx.begin() + q * 40,
                                                                   ridx.begin() + q * 40 + rcnt[q]);
    CHECK(same);
    double st[24];
    std::uint32_t kb = 0;
    CHECK(ref.evaluate(inst.queries.data(), n, inst.keys.data(), inst.values.data(), n, d,
                       inst.scale, inst.causal_offsets.data(), 0.05, mh.w1.data(), mh.b1.data(),
                       mh.w2.data(), d, L, est.projection.data(), r, st, &kb) == 0);
    CHECK(kb == rep.budget);
    for (int i = 0; i < 4; ++i) {
        const MethodReport& m = rep.methods[i];
        // IoU statistics are exact (bit-identical index sets); the output
        // errors follow the attention tolerance (fp32, <= 1e-5 max-abs)
        CHECK(m.mean_iou == st[i * 6] && m.p10_iou == st[i * 6 + 1] && m.p50_iou == st[i * 6 + 2] &&
              m.p90_iou == st[i * 6 + 3]);
        CHECK(std::fabs(m.mean_rel_err - st[i * 6 + 4]) <= 1e-5 + 1e-3 * st[i * 6 + 4]);
        CHECK(std::fabs(m.max_rel_err - st[i * 6 + 5]) <= 1e-5 + 1e-3 * st[i * 6 + 5]);
    }
}

TEST_CASE("oracle_topk: exact logits top-k, causal clamp, rejection; iou vs hash_topk") {
    std::mt19937_64 eng(77);
    const std::uint32_t n = 500, d = 64;
    AttentionInstance inst = make_causal_instance(random_matrix(n, d, eng), random_matrix(n, d, eng),
                                                  random_matrix(n, d, eng));
    const RetrievalResult o = oracle_topk(inst, 32);
    CHECK(o.method == RetrievalMethod::oracle);
    CHECK(o.indices[0].size() == 1 && o.indices[0][0] == 0);  // query 0 sees one row
    CHECK(o.indices[n - 1].size() == 32);
    CHECK(std::is_sorted(o.indices[n - 1].begin(), o.indices[n - 1].end()));
    CHECK_THROWS_AS(oracle_topk(inst, 0), DimensionError);
    const MlpHasher h = mlp_gaussian_init(d, d, 128, 64.0f, 5);
    const RetrievalResult r = hash_topk(inst, h, 32);
    for (std::uint32_t q = 0; q < n; q += 50) {
        const double v = iou(r.indices[q], o.indices[q]);
        CHECK(v >= 0.0 && v <= 1.0);
    }
    static Ref ref;
    if (!ref.h || !ref.oracle) return;
    std::vector<std::uint32_t> ridx(static_cast<std::size_t>(n) * 32), rcnt(n);
    CHECK(ref.oracle(inst.queries.data(), n, inst.keys.data(), n, d, inst.scale,
                     inst.causal_offsets.data(), 32, ridx.data(), rcnt.data()) == 0);
    bool same = true;
    for (std::uint32_t q = 0; q < n; ++q)
        same = same && o.indices[q] == std::vector<std::uint32_t>(ridx.begin() + q * 32,
                                                                  ridx.begin() + q * 32 + rcnt[q]);
    CHECK(same);
}

TEST_CASE("drop-in == reference: mlp_forward, hash_topk, sparse_attention") {
    static Ref ref;
    if (!ref.h) {
        std::fprintf(stderr, "note: oracle/_ref/libspotref.so not present, reference diff skipped\n");
        return;
    }
    std::mt19937_64 eng(2024);
    const std::uint32_t n = 600, d = 128, L = 128;
    const MlpHasher h = mlp_gaussian_init(d, d, L, 64.0f, 99);
    AttentionInstance inst = make_causal_instance(random_matrix(n, d, eng), random_matrix(n, d, eng),
                                                  random_matrix(n, d, eng));
    const Matrix<float> pre = mlp_forward(h, inst.keys);
    std::vector<float> rpre(pre.size());
    CHECK(ref.mlp_forward(h.w1.data(), h.b1.data(), h.w2.data(), d, d, L, inst.keys.data(), n,
                          rpre.data()) == 0);
    CHECK(std::memcmp(rpre.data(), pre.data(), pre.size() * 4) == 0);
    const std::uint32_t k = 24;
    const RetrievalResult res = hash_topk(inst, h, k);
    std::vector<std::uint32_t> ridx(static_cast<std::size_t>(n) * k), rcnt(n);
    CHECK(ref.hash_topk(h.w1.data(), h.b1.data(), h.w2.data(), d, L, inst.queries.data(), n,
                        inst.keys.data(), inst.values.data(), n, d, inst.scale,
                        inst.causal_offsets.data(), k, ridx.data(), rcnt.data()) == 0);
    bool same = true;
    for (std::uint32_t r = 0; r < n; ++r) {
        std::vector<std::uint32_t> want(ridx.begin() + static_cast<std::size_t>(r) * k,
                                        ridx.begin() + static_cast<std::size_t>(r) * k + rcnt[r]);
        if (same && res.indices[r] != want) {
            std::fprintf(stderr, "hash_topk differs at query %u (got %zu, want %zu):", r,
                         res.indices[r].size(), want.size());
            for (std::size_t i = 0; i < want.size() && i < res.indices[r].size(); ++i)
                if (res.indices[r][i] != want[i])
                    std::fprintf(stderr, " [%zu] %u!=%u", i, res.indices[r][i], want[i]);
            std::fprintf(stderr, "\n");
        }
        same = same && (res.indices[r] == want);
    }
    CHECK(same);
    const Matrix<float> sp = sparse_attention(inst, res);
    std::vector<std::uint32_t> flat;
    std::vector<std::uint64_t> off(n + 1, 0);
    for (std::uint32_t r = 0; r < n; ++r) {
        flat.insert(flat.end(), res.indices[r].begin(), res.indices[r].end());
        off[r + 1] = flat.size();
    }
    std::vector<float> rout(static_cast<std::size_t>(n) * d);
    CHECK(ref.sparse(inst.queries.data(), n, inst.keys.data(), inst.values.data(), n, d, inst.scale,
                     inst.causal_offsets.data(), flat.data(), off.data(), rout.data()) == 0);
    double mx = 0;
    for (std::size_t i = 0; i < rout.size(); ++i) mx = std::max(mx, (double)std::fabs(rout[i] - sp.data()[i]));
    std::fprintf(stderr, "sparse_attention max-abs vs reference: %.3g\n", mx);
    CHECK(mx <= 1e-5);
}

// ------------------------------------------------------------ trainer (§8 f4)
// The reference's test_trainer.cpp cases that exercise train_hasher through
// the public API (lr schedule, zero-lr identity, determinism, validation,
// loss trend on cone-shaped data), plus a bit-exact comparison with the
// reference's own train_hasher when oracle/_ref is present.
static TrainDataset cone_dataset(std::uint32_t n, std::uint32_t d, std::uint64_t seed) {
    // queries and keys share a common direction (a cone): retrieval is learnable
    std::mt19937_64 eng(seed);
    std::normal_distribution<double> g(0.0, 1.0);
    std::vector<double> axis(d);
    for (auto& a : axis) a = g(eng);
    TrainDataset ds;
    QkSequence seq{Matrix<float>(n, d), Matrix<float>(n, d)};
    for (std::uint32_t i = 0; i < n; ++i)
        for (std::uint32_t c = 0; c < d; ++c) {
            seq.queries(i, c) = static_cast<float>(0.8 * axis[c] + g(eng));
            seq.keys(i, c) = static_cast<float>(0.8 * axis[c] + g(eng));
        }
    ds.sequences.push_back(std::move(seq));
    return ds;
}

TEST_CASE("trainer: lr_at warmup then cosine; TrainConfig validation") {
    TrainConfig cfg;
    cfg.num_iters = 100;
    cfg.warmup_iters = 10;
    CHECK(lr_at(0, cfg) == 0.0);
    CHECK(std::fabs(lr_at(5, cfg) - 0.5e-3) < 1e-18);
    CHECK(lr_at(10, cfg) == cfg.max_lr);
    CHECK(std::fabs(lr_at(99, cfg) - cfg.min_lr) < 1e-18);
    TrainConfig bad = cfg;
    bad.min_lr = 1.0;
    CHECK_THROWS_AS(bad.validate(), DimensionError);
    bad = cfg;
    bad.batch = 0;
    CHECK_THROWS_AS(bad.validate(), DimensionError);
}

TEST_CASE("trainer: zero lr leaves the hasher bit-identical; runs are deterministic") {
    const TrainDataset ds = cone_dataset(160, 32, 5);
    RankingLossConfig rc;
    rc.maskout = 0.9;
    rc.max_oth = 32;
    rc.query_subsample = 16;
    TrainConfig cfg;
    cfg.num_iters = 4;
    cfg.warmup_iters = 2;
    cfg.holdout_queries = 16;
    const MlpHasher h0 = mlp_gaussian_init(32, 32, 32, 64.0f, 3);
    AnyHasher a = h0;
    TrainConfig z = cfg;
    z.max_lr = 0.0;
    const TrainReport r0 = train_hasher(a, ds, rc, z);
    const MlpHasher& az = std::get<MlpHasher>(a);
    CHECK(std::memcmp(az.w1.data(), h0.w1.data(), h0.w1.size() * 4) == 0);
    CHECK(std::memcmp(az.w2.data(), h0.w2.data(), h0.w2.size() * 4) == 0);
    CHECK(r0.records.size() == 4 && r0.skipped_steps == 0);
    AnyHasher b1 = h0, b2 = h0;
    const TrainReport ra = train_hasher(b1, ds, rc, cfg);
    const TrainReport rb = train_hasher(b2, ds, rc, cfg);
    CHECK(std::memcmp(std::get<MlpHasher>(b1).w1.data(), std::get<MlpHasher>(b2).w1.data(),
                      h0.w1.size() * 4) == 0);
    CHECK(format_train_report(ra, {}) == format_train_report(rb, {}));
    CHECK(std::memcmp(std::get<MlpHasher>(b1).w1.data(), h0.w1.data(), h0.w1.size() * 4) != 0);
}

TEST_CASE("trainer: input validation mirrors the reference") {
    RankingLossConfig rc;
    TrainConfig cfg;
    cfg.num_iters = 1;
    AnyHasher a = mlp_gaussian_init(16, 16, 32, 64.0f, 1);
    TrainDataset empty;
    CHECK_THROWS_WITH(train_hasher(a, empty, rc, cfg), DimensionError, "dataset is empty");
    TrainDataset mis;
    mis.sequences.push_back(QkSequence{Matrix<float>(8, 16), Matrix<float>(9, 16)});
    CHECK_THROWS_WITH(train_hasher(a, mis, rc, cfg), DimensionError, "causally aligned");
    TrainDataset wrong = cone_dataset(64, 8, 1);
    CHECK_THROWS_WITH(train_hasher(a, wrong, rc, cfg), DimensionError, "does not match hasher dimension");
    TrainDataset tiny = cone_dataset(20, 16, 1);  // floor(20 * 0.02) = 0 top keys
    CHECK_THROWS_WITH(train_hasher(a, tiny, rc, cfg), DimensionError, "top count floored to zero");
}

TEST_CASE("trainer: loss trends downward on cone data") {
    const TrainDataset ds = cone_dataset(512, 64, 17);
    RankingLossConfig rc;
    rc.max_oth = 64;
    rc.query_subsample = 32;
    TrainConfig cfg;
    cfg.num_iters = 200;
    cfg.warmup_iters = 10;
    cfg.max_lr = 3e-3;
    AnyHasher a = mlp_gaussian_init(64, 64, 64, 64.0f, 8);
    const TrainReport r = train_hasher(a, ds, rc, cfg);
    double first = 0, last = 0;
    for (int i = 0; i < 20; ++i) {
        first += r.records[i].loss;
        last += r.records[r.records.size() - 1 - i].loss;
    }
    std::fprintf(stderr, "trainer loss first20 %.4f last20 %.4f holdout IoU %.4f\n", first / 20,
                 last / 20, r.final_holdout_iou);
    CHECK(last < first);
}

TEST_CASE("trainer: drop-in == reference train_hasher (bit-identical weights)") {
    static Ref ref;
    if (!ref.h || !ref.train) {
        std::fprintf(stderr, "note: oracle/_ref/libspotref.so not present, reference diff skipped\n");
        return;
    }
    const TrainDataset ds = cone_dataset(300, 64, 23);
    RankingLossConfig rc;
    rc.max_oth = 48;
    rc.query_subsample = 20;
    TrainConfig cfg;
    cfg.num_iters = 12;
    cfg.warmup_iters = 3;
    cfg.seed = 77;
    cfg.holdout_queries = 40;
    MlpHasher h0 = mlp_gaussian_init(64, 96, 64, 64.0f, 12);
    AnyHasher a = h0;
    const TrainReport r = train_hasher(a, ds, rc, cfg);
    const double dc[12] = {cfg.max_lr, cfg.min_lr, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps,
                           cfg.weight_decay, cfg.grad_clip, cfg.soft_gamma, cfg.holdout_budget_rate,
                           rc.beta, rc.alpha, rc.maskout};
    const std::uint64_t uc[5] = {cfg.num_iters, cfg.warmup_iters, cfg.batch, cfg.seed,
                                 cfg.holdout_queries};
    const std::int64_t op[3] = {-1, 48, 20};
    std::vector<double> rec(3 * cfg.num_iters);
    double iou = 0;
    std::uint32_t sk = 0, len = 300;
    CHECK(ref.train(1, h0.w1.data(), h0.b1.data(), h0.w2.data(), 64, 96, 64, 64.0f, 1,
                    ds.sequences[0].queries.data(), ds.sequences[0].keys.data(), &len, dc, uc, op,
                    0, rec.data(), &iou, &sk) == 0);
    const MlpHasher& g = std::get<MlpHasher>(a);
    CHECK(std::memcmp(g.w1.data(), h0.w1.data(), h0.w1.size() * 4) == 0);
    CHECK(std::memcmp(g.b1.data(), h0.b1.data(), h0.b1.size() * 4) == 0);
    CHECK(std::memcmp(g.w2.data(), h0.w2.data(), h0.w2.size() * 4) == 0);
    CHECK(r.final_holdout_iou == iou);
    for (std::uint32_t i = 0; i < cfg.num_iters; ++i) {
        CHECK(r.records[i].lr == rec[3 * i + 2]);
        CHECK(r.records[i].violation_rate == rec[3 * i + 1]);
        CHECK(std::fabs(r.records[i].loss - rec[3 * i]) <= 1e-10 * std::fabs(rec[3 * i]));
    }
}

TEST_CASE("SPLQ dump round trip, validation and training from a dump") {
    std::mt19937_64 eng(4);
    const Matrix<float> q = random_matrix(120, 16, eng), k = random_matrix(120, 16, eng);
    const std::string path = "/tmp/spl_test_dump_" + std::to_string(::getpid()) + ".splq";
    write_dump(path, q, k);
    const QkDump d = read_dump(path);
    CHECK(d.queries.rows() == 120 && d.keys.cols() == 16);
    CHECK(std::memcmp(d.queries.data(), q.data(), q.size() * 4) == 0);
    CHECK(std::memcmp(d.keys.data(), k.data(), k.size() * 4) == 0);
    CHECK_THROWS_AS(write_dump(path, q, random_matrix(4, 8, eng)), DimensionError);
    Matrix<float> bad = q;
    bad.data()[3] = std::nanf("");
    CHECK_THROWS_AS(write_dump(path, bad, k), NumericError);
    {
        std::FILE* f = std::fopen(path.c_str(), "r+b");
        std::fseek(f, 0, SEEK_SET);
        std::fputc('X', f);
        std::fclose(f);
    }
    CHECK_THROWS_WITH(read_dump(path), FormatError, "bad magic");
    write_dump(path, q, k);
    TrainDataset ds = dataset_from_dump(read_dump(path));
    std::remove(path.c_str());
    RankingLossConfig rc;
    rc.maskout = 0.9;
    rc.max_oth = 16;
    rc.query_subsample = 8;
    TrainConfig cfg;
    cfg.num_iters = 3;
    cfg.holdout_queries = 16;
    AnyHasher a = mlp_gaussian_init(16, 16, 32, 64.0f, 2);
    const TrainReport r = train_hasher(a, ds, rc, cfg);
    CHECK(r.records.size() == 3);
    const std::string txt = format_train_report(r, std::vector<std::string>{"dump test"});
    CHECK(txt.rfind("# dump test\n# columns: iter loss violation_rate lr\n0 ", 0) == 0);
    CHECK(txt.find("# skipped_steps 0") != std::string::npos);
}

int main() {
    for (auto& [name, fn] : registry()) {
        g_case = name;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_failed;
            std::fprintf(stderr, "FAIL [%s] unexpected exception: %s\n", name, e.what());
        }
    }
    std::printf("%d checks, %d failed, %zu test cases\n", g_checks, g_failed, registry().size());
    return g_failed ? 1 : 0;
}
