// C++ drop-in of the reference's hot-path API (include/spotlight/*.hpp) on
// top of the C-ABI (include/spl_c.h). Host-side only: marshals host buffers
// to the device, calls the sm_100a kernels, copies results back and re-throws
// the reference's exception types with its wording. Every compute path is a
// GPU launch; without a Blackwell GPU the calls throw DeviceError.
//
// Concurrency: the reference functions are pure and thread-safe
// (SPEC.md:88-89); here each host thread gets its own spl_ctx (thread_local),
// which keeps that property.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <sstream>
#include <fstream>
#include <memory>
#include <random>
#include <string>
#include <type_traits>
#include <vector>

#include "spl_c.h"
#include <chrono>
#include <cstdio>

#include "spotlight/synthkv.hpp"
#include "spotlight/trainer.hpp"
#include "spotlight/attention_eval.hpp"
#include "spotlight/bitcodes.hpp"
#include "spotlight/hashers.hpp"

namespace spotlight {
namespace {

// ------------------------------------------------------------- plumbing
struct CtxHolder {
    spl_ctx* c = nullptr;
    ~CtxHolder() {
        if (c) spl_ctx_destroy(c);
    }
};

spl_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.c) {
        const char* dev = std::getenv("SPOTLIGHT_DEVICE");
        const spl_status st = spl_ctx_create(dev ? std::atoi(dev) : 0, &h.c);
        if (st != SPL_OK) {
            h.c = nullptr;
            throw DeviceError("spotlight: no usable sm_100 GPU (spl_ctx_create failed)");
        }
    }
    return h.c;
}

[[noreturn]] void raise(spl_status st) {
    const std::string msg = spl_last_error(ctx());
    switch (st) {
        case SPL_E_DIMENSION: throw DimensionError(msg);
        case SPL_E_NUMERIC: throw NumericError(msg);
        case SPL_E_FORMAT: throw FormatError(msg);
        case SPL_E_IO: throw IoError(msg);
        case SPL_E_EMPTY_PAIRS: throw EmptyPairError(msg);
        default: throw DeviceError(msg.empty() ? "spotlight: device failure" : msg);
    }
}

void check(spl_status st) {
    if (st != SPL_OK) raise(st);
}

// Synchronise the (default) stream and surface device-side error words.
void finish() {
    check(spl_stream_synchronize(ctx(), nullptr));
    check(spl_check_device_error(ctx(), nullptr));
}

class DevBuf {
public:
    explicit DevBuf(std::size_t bytes) : n_(bytes) { check(spl_device_alloc(ctx(), bytes ? bytes : 4, &p_)); }
    DevBuf(const void* host, std::size_t bytes) : DevBuf(bytes) { upload(host, bytes); }
    ~DevBuf() {
        if (p_) spl_device_free(ctx(), p_);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    void upload(const void* host, std::size_t bytes) {
        if (bytes) check(spl_memcpy(ctx(), p_, host, bytes, nullptr));
    }
    void download(void* host, std::size_t bytes) const {
        if (bytes) check(spl_memcpy(ctx(), host, p_, bytes, nullptr));
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p_);
    }

private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
};

// A device hasher bank of one head for the duration of a call.
class DevHasher {
public:
    explicit DevHasher(const MlpHasher& h) {
        if (h.w2.rows() != h.w1.cols() || h.b1.size() != h.w1.cols())
            throw DimensionError("mlp_forward: inconsistent hasher shapes");
        check(spl_hasher_create(ctx(), SPL_HASHER_MLP, 1, h.input_dim(), h.hidden_dim(),
                                h.code_bits(), h.w1.data(), h.b1.data(), h.w2.data(), &h_));
    }
    explicit DevHasher(const LinearHasher& h) {
        check(spl_hasher_create(ctx(), SPL_HASHER_LINEAR, 1, h.input_dim(), 0, h.code_bits(),
                                h.projection.data(), nullptr, nullptr, &h_));
    }
    ~DevHasher() { spl_hasher_destroy(h_); }
    DevHasher(const DevHasher&) = delete;
    DevHasher& operator=(const DevHasher&) = delete;
    const spl_hasher* get() const { return h_; }

private:
    spl_hasher* h_ = nullptr;
};

// Codes of x (m x d) through the GPU exact encoder, as a host CodeMatrix.
template <typename H>
CodeMatrix encode_codes(const H& hasher, const Matrix<float>& x, std::uint32_t L) {
    CodeMatrix out(static_cast<std::uint32_t>(x.rows()), L);
    if (x.rows() == 0) return out;
    DevHasher dh(hasher);
    DevBuf dx(x.data(), x.size() * sizeof(float));
    DevBuf dc(out.raw().size() * 4);
    check(spl_encode(ctx(), dh.get(), dx.as<float>(), 1, static_cast<std::uint32_t>(x.rows()),
                     SPL_ENCODE_EXACT, dc.as<std::uint32_t>(), nullptr));
    finish();
    dc.download(out.raw().data(), out.raw().size() * 4);
    return out;
}

std::string str(std::size_t v) { return std::to_string(v); }

// ------------------------------------------------------------- little-endian file I/O
void write_u32(std::ofstream& os, std::uint32_t v) {
    const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                                static_cast<unsigned char>(v >> 16),
                                static_cast<unsigned char>(v >> 24)};
    os.write(reinterpret_cast<const char*>(b), 4);
}
void write_f32(std::ofstream& os, float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    write_u32(os, u);
}
template <typename T>
void write_words(std::ofstream& os, const T* p, std::size_t n) {
    static_assert(sizeof(T) == 4);
    for (std::size_t i = 0; i < n; ++i) {
        std::uint32_t u;
        std::memcpy(&u, p + i, 4);
        write_u32(os, u);
    }
}

class Reader {
public:
    explicit Reader(const std::string& path) : path_(path), is_(path, std::ios::binary) {
        if (!is_) throw IoError("cannot open for reading: " + path);
    }
    void magic(const char* m) {
        char got[4];
        if (!is_.read(got, 4)) throw FormatError(path_ + ": truncated while reading magic at offset 0");
        if (std::memcmp(got, m, 4) != 0)
            throw FormatError(path_ + ": bad magic at offset 0, expected \"" + std::string(m, 4) +
                              "\" got \"" + std::string(got, 4) + "\"");
    }
    std::uint32_t u32(const char* field) {
        unsigned char b[4];
        // the offset is the stream position after the failed read, as the
        // reference reports it (binary_io.hpp:36-41): tellg() of a failed
        // stream, i.e. -1
        if (!is_.read(reinterpret_cast<char*>(b), 4))
            throw FormatError(path_ + ": truncated while reading " + field + " at offset " +
                              std::to_string(static_cast<long long>(is_.tellg())));
        return b[0] | (b[1] << 8) | (b[2] << 16) | (static_cast<std::uint32_t>(b[3]) << 24);
    }
    std::uint8_t u8(const char* field) {
        char c;
        if (!is_.read(&c, 1)) throw FormatError(path_ + ": truncated while reading " + field);
        return static_cast<std::uint8_t>(c);
    }
    float f32(const char* field) {
        const std::uint32_t u = u32(field);
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    }
    template <typename T>
    void words(T* out, std::size_t n, const char* field) {
        static_assert(sizeof(T) == 4);
        std::vector<unsigned char> buf(n * 4);
        if (n && !is_.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(n * 4)))
            throw FormatError(path_ + ": truncated payload while reading " + field + " (expected " +
                              str(n * 4) + " bytes)");
        for (std::size_t i = 0; i < n; ++i) {
            const std::uint32_t u = buf[4 * i] | (buf[4 * i + 1] << 8) | (buf[4 * i + 2] << 16) |
                                    (static_cast<std::uint32_t>(buf[4 * i + 3]) << 24);
            std::memcpy(out + i, &u, 4);
        }
    }

private:
    std::string path_;
    std::ifstream is_;
};

std::ofstream open_out(const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open for writing: " + path);
    return os;
}

}  // namespace

// =================================================================== bitcodes
CodeMatrix::CodeMatrix(std::uint32_t rows, std::uint32_t length_bits) : n_(rows), L_(length_bits) {
    if (length_bits == 0 || length_bits % 32 != 0)
        throw DimensionError("CodeMatrix: length_bits " + str(length_bits) +
                             " must be a positive multiple of 32");
    if (length_bits > kMaxBits)
        throw DimensionError("CodeMatrix: length_bits " + str(length_bits) + " exceeds the " +
                             str(kMaxBits) + "-bit limit");
    w_.assign(static_cast<std::size_t>(rows) * (length_bits / 32), 0u);
}

CodeMatrix pack_bits(const BitMatrix& bits) {
    const std::size_t d = bits.cols();
    if (d == 0 || d % 32 != 0)
        throw DimensionError("pack_bits: column count " + str(d) + " must be a positive multiple of 32");
    CodeMatrix out(static_cast<std::uint32_t>(bits.rows()), static_cast<std::uint32_t>(d));
    if (bits.rows() == 0) return out;
    DevBuf db(bits.data(), bits.rows() * d);
    DevBuf dc(out.raw().size() * 4);
    check(spl_pack_bits(ctx(), db.as<std::uint8_t>(), bits.rows(), static_cast<std::uint32_t>(d),
                        dc.as<std::uint32_t>(), nullptr));
    finish();
    dc.download(out.raw().data(), out.raw().size() * 4);
    return out;
}

BitMatrix unpack_bits(const CodeMatrix& codes) {
    BitMatrix out(codes.rows(), codes.length_bits());
    if (codes.rows() == 0) return out;
    DevBuf dc(codes.raw().data(), codes.raw().size() * 4);
    DevBuf db(static_cast<std::size_t>(codes.rows()) * codes.length_bits());
    check(spl_unpack_bits(ctx(), dc.as<std::uint32_t>(), codes.rows(), codes.length_bits(),
                          db.as<std::uint8_t>(), nullptr));
    finish();
    db.download(out.data(), static_cast<std::size_t>(codes.rows()) * codes.length_bits());
    return out;
}

void nxor_scores_into(std::span<const std::uint32_t> query_words, const CodeMatrix& index,
                      std::uint32_t n_valid, std::int32_t* out) {
    const std::size_t wpr = index.words_per_row();
    if (query_words.size() != wpr)
        throw DimensionError("nxor_scores: query has " + str(query_words.size() * 32) +
                             " bits, index has " + str(index.length_bits()));
    if (n_valid == 0) return;
    n_valid = std::min(n_valid, index.rows());
    DevBuf dc(index.raw().data(), static_cast<std::size_t>(n_valid) * wpr * 4);
    DevBuf dq(query_words.data(), wpr * 4);
    DevBuf dn(&n_valid, 4);
    DevBuf ds(static_cast<std::size_t>(n_valid) * 4);
    check(spl_nxor_scores(ctx(), dc.as<std::uint32_t>(), 0, index.length_bits(),
                          dq.as<std::uint32_t>(), 1, dn.as<std::uint32_t>(), 1, n_valid,
                          ds.as<std::int32_t>(), n_valid, nullptr));
    finish();
    ds.download(out, static_cast<std::size_t>(n_valid) * 4);
}

ScoreVector nxor_scores(const HashCode& query, const CodeMatrix& index) {
    if (query.length_bits != index.length_bits())
        throw DimensionError("nxor_scores: query length " + str(query.length_bits) +
                             " != index length " + str(index.length_bits()));
    ScoreVector s(index.rows());
    nxor_scores_into(std::span<const std::uint32_t>(query.words.data(), query.words.size()), index,
                     index.rows(), s.data());
    return s;
}

template <typename S>
std::vector<std::uint32_t> top_k_indices(std::span<const S> scores, std::uint32_t k) {
    const std::size_t n = scores.size();
    if (k == 0 || k > n)
        throw DimensionError("top_k_indices: k=" + str(k) + " out of range for n=" + str(n));
    constexpr int dtype = std::is_same_v<S, std::int32_t> ? 0 : (std::is_same_v<S, float> ? 1 : 2);
    DevBuf ds(scores.data(), n * sizeof(S));
    DevBuf di(static_cast<std::size_t>(k) * 4);
    check(spl_top_k(ctx(), ds.as<void>(), dtype, 1, n, n, k, di.as<std::uint32_t>(), nullptr));
    finish();
    std::vector<std::uint32_t> out(k);
    di.download(out.data(), static_cast<std::size_t>(k) * 4);
    return out;
}

template std::vector<std::uint32_t> top_k_indices<std::int32_t>(std::span<const std::int32_t>,
                                                                std::uint32_t);
template std::vector<std::uint32_t> top_k_indices<float>(std::span<const float>, std::uint32_t);
template std::vector<std::uint32_t> top_k_indices<double>(std::span<const double>, std::uint32_t);

void write_code_index(const std::string& path, const CodeMatrix& codes) {
    auto os = open_out(path);
    os.write("SPLC", 4);
    write_u32(os, 1);
    write_u32(os, codes.rows());
    write_u32(os, codes.length_bits());
    write_words(os, codes.raw().data(), codes.raw().size());
    if (!os) throw IoError("write failed: " + path);
}

CodeMatrix read_code_index(const std::string& path) {
    Reader r(path);
    r.magic("SPLC");
    const std::uint32_t version = r.u32("version");
    if (version != 1) throw FormatError(path + ": unsupported SPLC version " + str(version));
    const std::uint32_t n = r.u32("row count");
    const std::uint32_t bits = r.u32("code length");
    CodeMatrix codes(n, bits);
    r.words(codes.raw().data(), codes.raw().size(), "code words");
    return codes;
}

// ==================================================================== hashers
MlpHasher mlp_gaussian_init(std::uint32_t d, std::uint32_t h, std::uint32_t code_bits,
                            float gamma, std::uint64_t seed) {
    if (d < 1 || h < 1 || code_bits < 1)
        throw DimensionError("mlp_gaussian_init: dimensions must be >= 1");
    if (gamma <= 0.0f) throw DimensionError("mlp_gaussian_init: gamma must be positive");
    // The same engine and distribution (mt19937_64, normal_distribution<double>)
    // in the same draw order: W1 row-major, then W2 row-major.
    std::mt19937_64 eng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    MlpHasher m;
    m.w1 = Matrix<float>(d, h);
    const double s1 = 1.0 / std::sqrt(static_cast<double>(d));
    for (std::size_t i = 0; i < m.w1.size(); ++i) m.w1.data()[i] = static_cast<float>(gauss(eng) * s1);
    m.b1.assign(h, 0.0f);
    m.w2 = Matrix<float>(h, code_bits);
    const double s2 = 1.0 / std::sqrt(static_cast<double>(h));
    for (std::size_t i = 0; i < m.w2.size(); ++i) m.w2.data()[i] = static_cast<float>(gauss(eng) * s2);
    m.gamma = gamma;
    return m;
}

namespace {

// Code widths the exact encoder takes: whole 32-bit words. Wider layer-2 /
// projection copies with zero columns give the same pre-activations for the
// real columns (each column is its own FMA chain); the extra ones are dropped.
std::uint32_t padded_bits(std::size_t L) { return static_cast<std::uint32_t>((L + 31) / 32 * 32); }

Matrix<float> pad_cols(const Matrix<float>& m, std::size_t cols) {
    if (m.cols() == cols) return m;
    Matrix<float> out(m.rows(), cols);
    for (std::size_t i = 0; i < m.rows(); ++i)
        std::copy(m.row(i).begin(), m.row(i).end(), out.row(i).begin());
    return out;
}

template <typename T>
void require_finite(const Matrix<T>& m, const char* what) {
    if (!m.all_finite()) throw NumericError(std::string(what) + " contains non-finite values");
}

// The double instances: spl_matmul / spl_map on device buffers.
template <typename T>
constexpr int dtype_of() {
    return std::is_same_v<T, double> ? SPL_F64 : SPL_F32;
}

template <typename T>
void device_matmul(const void* a, std::size_t m, std::size_t k, const void* b, std::size_t n, void* c) {
    check(spl_matmul(ctx(), dtype_of<T>(), a, m, k, b, n, c, nullptr));
}

template <typename T>
void check_mm(const Matrix<T>& a, const Matrix<T>& b) {
    if (a.cols() != b.rows())
        throw DimensionError("matmul: inner dimensions " + std::to_string(a.cols()) + " and " +
                             std::to_string(b.rows()) + " do not match");
}

// pre-activations of an f64 MLP hasher, left on the device
template <typename T>
DevBuf mlp_forward_dev(const MlpHasherT<T>& h, const Matrix<T>& x) {
    const std::size_t m = x.rows(), d = h.w1.rows(), hd = h.w1.cols(), L = h.w2.cols();
    DevBuf dx(x.data(), x.size() * sizeof(T)), dw1(h.w1.data(), h.w1.size() * sizeof(T));
    DevBuf db1(h.b1.data(), h.b1.size() * sizeof(T)), dw2(h.w2.data(), h.w2.size() * sizeof(T));
    DevBuf z1(m * hd * sizeof(T)), z2(m * L * sizeof(T));
    device_matmul<T>(dx.as<void>(), m, d, dw1.as<void>(), hd, z1.as<void>());
    check(spl_map(ctx(), dtype_of<T>(), SPL_MAP_BIAS_SILU, z1.as<void>(), m, hd, db1.as<void>(), 0.0,
                  z1.as<void>(), nullptr));
    device_matmul<T>(z1.as<void>(), m, hd, dw2.as<void>(), L, z2.as<void>());
    return z2;
}

template <typename T>
void mlp_checks(const MlpHasherT<T>& h, const Matrix<T>& x) {
    if (x.cols() != h.w1.rows())
        throw DimensionError("mlp_forward: input dim " + str(x.cols()) + " != hasher dim " +
                             str(h.w1.rows()));
    if (h.w2.rows() != h.w1.cols() || h.b1.size() != h.w1.cols())
        throw DimensionError("mlp_forward: inconsistent hasher shapes");
    require_finite(h.w1, "mlp w1");
    require_finite(h.w2, "mlp w2");
    for (const T& v : h.b1)
        if (!std::isfinite(static_cast<double>(v))) throw NumericError("mlp b1 is non-finite");
    require_finite(x, "mlp input");
}

template <typename T>
BitMatrix sign_bits_dev(const DevBuf& pre, std::size_t m, std::size_t L) {
    BitMatrix bits(m, L);
    if (m == 0 || L == 0) return bits;
    DevBuf db(m * L);
    check(spl_map(ctx(), dtype_of<T>(), SPL_MAP_SIGN_BITS, pre.as<void>(), m, L, nullptr, 0.0,
                  db.as<void>(), nullptr));
    finish();
    db.download(bits.data(), m * L);
    return bits;
}

}  // namespace

template <typename T>
Matrix<T> matmul(const Matrix<T>& a, const Matrix<T>& b) {
    check_mm(a, b);
    Matrix<T> c(a.rows(), b.cols());
    if (c.size() == 0) return c;
    DevBuf da(a.data(), a.size() * sizeof(T)), dbm(b.data(), b.size() * sizeof(T)), dc(c.size() * sizeof(T));
    device_matmul<T>(da.as<void>(), a.rows(), a.cols(), dbm.as<void>(), b.cols(), dc.as<void>());
    finish();
    dc.download(c.data(), c.size() * sizeof(T));
    return c;
}
template Matrix<float> matmul<float>(const Matrix<float>&, const Matrix<float>&);
template Matrix<double> matmul<double>(const Matrix<double>&, const Matrix<double>&);

template <typename T>
Matrix<T> mlp_forward(const MlpHasherT<T>& h, const Matrix<T>& x) {
    if constexpr (std::is_same_v<T, float>) {
        if (x.cols() != h.w1.rows())
            throw DimensionError("mlp_forward: input dim " + str(x.cols()) + " != hasher dim " +
                                 str(h.w1.rows()));
        Matrix<float> pre(x.rows(), h.code_bits());
        if (x.rows() == 0 || h.code_bits() == 0) return pre;
        const std::uint32_t Lp = padded_bits(h.code_bits());
        MlpHasher hp = h;
        hp.w2 = pad_cols(h.w2, Lp);
        DevHasher dh(hp);  // require_finite on the weights (spl_hasher_create)
        DevBuf dx(x.data(), x.size() * 4);
        DevBuf dp((std::size_t)x.rows() * Lp * 4);
        check(spl_mlp_forward(ctx(), dh.get(), dx.as<float>(), 1, static_cast<std::uint32_t>(x.rows()),
                              dp.as<float>(), nullptr));
        finish();
        if (Lp == h.code_bits()) {
            dp.download(pre.data(), pre.size() * 4);
        } else {
            Matrix<float> full(x.rows(), Lp);
            dp.download(full.data(), full.size() * 4);
            for (std::size_t i = 0; i < x.rows(); ++i)
                std::copy(full.row(i).begin(), full.row(i).begin() + h.code_bits(), pre.row(i).begin());
        }
        return pre;
    } else {
        mlp_checks(h, x);
        Matrix<T> pre(x.rows(), h.code_bits());
        if (pre.size() == 0) return pre;
        DevBuf z2 = mlp_forward_dev(h, x);
        finish();
        z2.download(pre.data(), pre.size() * sizeof(T));
        return pre;
    }
}
template Matrix<float> mlp_forward<float>(const MlpHasherT<float>&, const Matrix<float>&);
template Matrix<double> mlp_forward<double>(const MlpHasherT<double>&, const Matrix<double>&);

CodeMatrix mlp_hash_packed(const MlpHasher& h, const Matrix<float>& x) {
    if (x.cols() != h.w1.rows())
        throw DimensionError("mlp_forward: input dim " + str(x.cols()) + " != hasher dim " +
                             str(h.w1.rows()));
    return encode_codes(h, x, h.code_bits());
}

CodeMatrix linear_hash_packed(const LinearHasher& h, const Matrix<float>& x) {
    if (x.cols() != h.projection.rows())
        throw DimensionError("linear_hash: input dim " + str(x.cols()) + " != hasher dim " +
                             str(h.projection.rows()));
    return encode_codes(h, x, h.code_bits());
}

namespace {
// the first L columns of a padded-width code
BitMatrix first_cols(const BitMatrix& b, std::size_t L) {
    if (b.cols() == L) return b;
    BitMatrix out(b.rows(), L);
    for (std::size_t i = 0; i < b.rows(); ++i)
        std::copy(b.row(i).begin(), b.row(i).begin() + L, out.row(i).begin());
    return out;
}
}  // namespace

template <typename T>
BitMatrix mlp_hash(const MlpHasherT<T>& h, const Matrix<T>& x) {
    if constexpr (std::is_same_v<T, float>) {
        if (x.cols() != h.w1.rows())
            throw DimensionError("mlp_forward: input dim " + str(x.cols()) + " != hasher dim " +
                                 str(h.w1.rows()));
        if (x.rows() == 0 || h.code_bits() == 0) return BitMatrix(x.rows(), h.code_bits());
        MlpHasher hp = h;
        hp.w2 = pad_cols(h.w2, padded_bits(h.code_bits()));
        return first_cols(unpack_bits(encode_codes(hp, x, padded_bits(h.code_bits()))), h.code_bits());
    } else {
        mlp_checks(h, x);
        if (x.rows() == 0 || h.code_bits() == 0) return BitMatrix(x.rows(), h.code_bits());
        DevBuf z2 = mlp_forward_dev(h, x);
        return sign_bits_dev<T>(z2, x.rows(), h.code_bits());
    }
}
template BitMatrix mlp_hash<float>(const MlpHasherT<float>&, const Matrix<float>&);
template BitMatrix mlp_hash<double>(const MlpHasherT<double>&, const Matrix<double>&);

template <typename T>
BitMatrix linear_hash(const LinearHasherT<T>& h, const Matrix<T>& x) {
    if (x.cols() != h.projection.rows())
        throw DimensionError("linear_hash: input dim " + str(x.cols()) + " != hasher dim " +
                             str(h.projection.rows()));
    if (x.rows() == 0 || h.code_bits() == 0) return BitMatrix(x.rows(), h.code_bits());
    if constexpr (std::is_same_v<T, float>) {
        LinearHasher hp{pad_cols(h.projection, padded_bits(h.code_bits()))};
        return first_cols(unpack_bits(encode_codes(hp, x, padded_bits(h.code_bits()))), h.code_bits());
    } else {
        require_finite(h.projection, "linear projection");
        require_finite(x, "linear input");
        const std::size_t m = x.rows(), L = h.code_bits();
        DevBuf dx(x.data(), x.size() * sizeof(T)), dp(h.projection.data(), h.projection.size() * sizeof(T));
        DevBuf pre(m * L * sizeof(T));
        device_matmul<T>(dx.as<void>(), m, x.cols(), dp.as<void>(), L, pre.as<void>());
        return sign_bits_dev<T>(pre, m, L);
    }
}
template BitMatrix linear_hash<float>(const LinearHasherT<float>&, const Matrix<float>&);
template BitMatrix linear_hash<double>(const LinearHasherT<double>&, const Matrix<double>&);

template <typename T>
Matrix<T> soft_sign(const Matrix<T>& z, T gamma) {
    if (!(gamma > T(0))) throw DimensionError("soft_sign: gamma must be positive");
    Matrix<T> out(z.rows(), z.cols());
    if (out.size() == 0) return out;
    DevBuf dz(z.data(), z.size() * sizeof(T));
    check(spl_map(ctx(), dtype_of<T>(), SPL_MAP_SOFT_SIGN, dz.as<void>(), z.rows(), z.cols(), nullptr,
                  static_cast<double>(gamma), dz.as<void>(), nullptr));
    finish();
    dz.download(out.data(), out.size() * sizeof(T));
    return out;
}
template Matrix<float> soft_sign<float>(const Matrix<float>&, float);
template Matrix<double> soft_sign<double>(const Matrix<double>&, double);

template <typename T>
Matrix<T> soft_codes(const MlpHasherT<T>& h, const Matrix<T>& x) {
    return soft_sign(mlp_forward(h, x), h.gamma);
}
template Matrix<float> soft_codes<float>(const MlpHasherT<float>&, const Matrix<float>&);
template Matrix<double> soft_codes<double>(const MlpHasherT<double>&, const Matrix<double>&);

template <typename T>
std::vector<T> downproj_scores(const DownProjEstimatorT<T>& e, std::span<const T> q,
                               const Matrix<T>& keys) {
    const std::size_t d = e.projection.rows(), r = e.projection.cols(), n = keys.rows();
    if (q.size() != d || keys.cols() != d) throw DimensionError("downproj_scores: shape mismatch");
    std::vector<T> scores(n);
    if (n == 0) return scores;
    if (r == 0) return scores;
    // qp = q P and kp = K P (the reference's per-output FMA order), then
    // score_i = kp_i . qp: kp (n x r) times qp as an r x 1 matrix
    DevBuf dq(q.data(), d * sizeof(T)), dP(e.projection.data(), e.projection.size() * sizeof(T));
    DevBuf dk(keys.data(), keys.size() * sizeof(T)), qp(r * sizeof(T)), kp(n * r * sizeof(T));
    DevBuf ds(n * sizeof(T));
    device_matmul<T>(dq.as<void>(), 1, d, dP.as<void>(), r, qp.as<void>());
    device_matmul<T>(dk.as<void>(), n, d, dP.as<void>(), r, kp.as<void>());
    device_matmul<T>(kp.as<void>(), n, r, qp.as<void>(), 1, ds.as<void>());
    finish();
    ds.download(scores.data(), n * sizeof(T));
    return scores;
}
template std::vector<float> downproj_scores<float>(const DownProjEstimatorT<float>&, std::span<const float>,
                                                   const Matrix<float>&);
template std::vector<double> downproj_scores<double>(const DownProjEstimatorT<double>&, std::span<const double>,
                                                     const Matrix<double>&);

void write_hasher(const std::string& path, const AnyHasher& hasher) {
    auto os = open_out(path);
    os.write("SPLH", 4);
    write_u32(os, 1);
    if (const auto* lin = std::get_if<LinearHasher>(&hasher)) {
        os.put(0);
        write_u32(os, lin->input_dim());
        write_u32(os, 0);
        write_u32(os, lin->code_bits());
        write_f32(os, 0.0f);
        write_words(os, lin->projection.data(), lin->projection.size());
    } else if (const auto* mlp = std::get_if<MlpHasher>(&hasher)) {
        os.put(1);
        write_u32(os, mlp->input_dim());
        write_u32(os, mlp->hidden_dim());
        write_u32(os, mlp->code_bits());
        write_f32(os, mlp->gamma);
        write_words(os, mlp->w1.data(), mlp->w1.size());
        write_words(os, mlp->b1.data(), mlp->b1.size());
        write_words(os, mlp->w2.data(), mlp->w2.size());
    } else {
        const auto& dp = std::get<DownProjEstimator>(hasher);
        os.put(2);
        write_u32(os, dp.input_dim());
        write_u32(os, 0);
        write_u32(os, dp.reduced_dim());
        write_f32(os, 0.0f);
        write_words(os, dp.projection.data(), dp.projection.size());
    }
    if (!os) throw IoError("write failed: " + path);
}

AnyHasher read_hasher(const std::string& path) {
    Reader r(path);
    r.magic("SPLH");
    const std::uint32_t version = r.u32("version");
    if (version != 1) throw FormatError(path + ": unsupported SPLH version " + str(version));
    const std::uint8_t kind = r.u8("kind");
    const std::uint32_t d = r.u32("d"), h = r.u32("h"), L = r.u32("L");
    const float gamma = r.f32("gamma");
    auto mat = [&](std::size_t rows, std::size_t cols, const char* f) {
        Matrix<float> m(rows, cols);
        r.words(m.data(), m.size(), f);
        return m;
    };
    switch (kind) {
        case 0: return LinearHasher{mat(d, L, "projection")};
        case 1: {
            MlpHasher m;
            m.w1 = mat(d, h, "w1");
            m.b1.assign(h, 0.0f);
            r.words(m.b1.data(), m.b1.size(), "b1");
            m.w2 = mat(h, L, "w2");
            m.gamma = gamma;
            if (m.gamma <= 0.0f) throw FormatError(path + ": mlp gamma must be positive");
            return m;
        }
        case 2: return DownProjEstimator{mat(d, L, "projection")};
        default: throw FormatError(path + ": unknown hasher kind " + str(kind));
    }
}

const char* hasher_kind_name(const AnyHasher& hasher) {
    if (std::holds_alternative<LinearHasher>(hasher)) return "linear";
    if (std::holds_alternative<MlpHasher>(hasher)) return "mlp";
    return "downproj";
}

// ============================================================= attention_eval
void AttentionInstance::validate() const {
    const std::size_t n = keys.rows();
    if (n == 0) throw DimensionError("attention: empty KV cache");
    if (values.rows() != n) throw DimensionError("attention: key/value row counts differ");
    if (queries.cols() != keys.cols() || values.cols() != keys.cols())
        throw DimensionError("attention: embedding dimensions differ");
    if (!(scale > 0.0f)) throw DimensionError("attention: scale must be positive");
    if (causal_offsets.size() != queries.rows())
        throw DimensionError("attention: need one causal offset per query");
    for (std::uint32_t off : causal_offsets)
        if (off == 0 || off > n)
            throw DimensionError("attention: causal offset " + str(off) + " outside [1, " + str(n) + "]");
}

AttentionInstance make_causal_instance(Matrix<float> queries, Matrix<float> keys,
                                       Matrix<float> values) {
    if (queries.rows() != keys.rows())
        throw DimensionError("make_causal_instance: query count must equal cache size");
    AttentionInstance inst;
    inst.scale = 1.0f / std::sqrt(static_cast<float>(keys.cols()));
    inst.causal_offsets.resize(queries.rows());
    for (std::size_t i = 0; i < queries.rows(); ++i)
        inst.causal_offsets[i] = static_cast<std::uint32_t>(i + 1);
    inst.queries = std::move(queries);
    inst.keys = std::move(keys);
    inst.values = std::move(values);
    inst.validate();
    return inst;
}

const char* retrieval_method_name(RetrievalMethod m) {
    switch (m) {
        case RetrievalMethod::oracle: return "oracle";
        case RetrievalMethod::lsh: return "lsh";
        case RetrievalMethod::mlp: return "mlp";
        case RetrievalMethod::downproj: return "downproj";
    }
    return "?";
}

RetrievalResult hash_topk(const AttentionInstance& inst, const AnyHasher& hasher,
                          std::uint32_t k) {
    inst.validate();
    if (k == 0) throw DimensionError("hash_topk: k must be >= 1");
    if (std::holds_alternative<DownProjEstimator>(hasher))
        throw DimensionError("hash_topk: down-projection estimator is not a hash; use downproj_topk");
    const bool is_mlp = std::holds_alternative<MlpHasher>(hasher);
    const std::uint32_t dim = is_mlp ? std::get<MlpHasher>(hasher).input_dim()
                                     : std::get<LinearHasher>(hasher).input_dim();
    if (inst.keys.cols() != dim) throw DimensionError("hash_topk: hasher dimension mismatch");
    // Encode the whole cache and the queries once (K1), then one K3 launch
    // retrieves for every query against the shared code cache (stride 0),
    // query r seeing rows [0, causal_offsets[r]).
    const CodeMatrix key_codes = is_mlp ? mlp_hash_packed(std::get<MlpHasher>(hasher), inst.keys)
                                        : linear_hash_packed(std::get<LinearHasher>(hasher), inst.keys);
    const CodeMatrix query_codes = is_mlp
                                       ? mlp_hash_packed(std::get<MlpHasher>(hasher), inst.queries)
                                       : linear_hash_packed(std::get<LinearHasher>(hasher), inst.queries);
    const auto q = static_cast<std::uint32_t>(inst.num_queries());
    const auto n = static_cast<std::uint32_t>(inst.cache_size());
    RetrievalResult res;
    res.method = is_mlp ? RetrievalMethod::mlp : RetrievalMethod::lsh;
    res.budget = k;
    res.indices.resize(q);
    if (q == 0) return res;
    DevBuf dk(key_codes.raw().data(), key_codes.raw().size() * 4);
    DevBuf dq(query_codes.raw().data(), query_codes.raw().size() * 4);
    DevBuf dn(inst.causal_offsets.data(), static_cast<std::size_t>(q) * 4);
    DevBuf di(static_cast<std::size_t>(q) * k * 4);
    DevBuf dc(static_cast<std::size_t>(q) * 4);
    check(spl_hamming_topk(ctx(), dk.as<std::uint32_t>(), 0, key_codes.length_bits(),
                           dq.as<std::uint32_t>(), q, dn.as<std::uint32_t>(), 1, n, k,
                           di.as<std::uint32_t>(), dc.as<std::uint32_t>(), nullptr));
    finish();
    std::vector<std::uint32_t> idx(static_cast<std::size_t>(q) * k), cnt(q);
    di.download(idx.data(), idx.size() * 4);
    dc.download(cnt.data(), cnt.size() * 4);
    for (std::uint32_t r = 0; r < q; ++r)
        res.indices[r].assign(idx.begin() + static_cast<std::size_t>(r) * k,
                              idx.begin() + static_cast<std::size_t>(r) * k + cnt[r]);
    return res;
}

namespace {
// Exact dense top-k of q x d queries against n x d keys (shared by all
// queries, causal offsets per query) on the GPU: spl_oracle_topk.
std::vector<std::vector<std::uint32_t>> dense_topk(const float* queries, std::uint32_t q,
                                                   const float* keys, std::uint32_t n,
                                                   std::uint32_t d, const std::uint32_t* offsets,
                                                   float scale, std::uint32_t k) {
    std::vector<std::vector<std::uint32_t>> out(q);
    if (q == 0) return out;
    DevBuf dqv(queries, static_cast<std::size_t>(q) * d * 4);
    DevBuf dkv(keys, static_cast<std::size_t>(n) * d * 4);
    DevBuf dn(offsets, static_cast<std::size_t>(q) * 4);
    DevBuf di(static_cast<std::size_t>(q) * k * 4);
    DevBuf dc(static_cast<std::size_t>(q) * 4);
    check(spl_oracle_topk(ctx(), dqv.as<float>(), dkv.as<float>(), SPL_F32, 0, d, q,
                          dn.as<std::uint32_t>(), 1, n, scale, k, di.as<std::uint32_t>(),
                          dc.as<std::uint32_t>(), nullptr, nullptr));
    finish();
    std::vector<std::uint32_t> idx(static_cast<std::size_t>(q) * k), cnt(q);
    di.download(idx.data(), idx.size() * 4);
    dc.download(cnt.data(), cnt.size() * 4);
    for (std::uint32_t r = 0; r < q; ++r)
        out[r].assign(idx.begin() + static_cast<std::size_t>(r) * k,
                      idx.begin() + static_cast<std::size_t>(r) * k + cnt[r]);
    return out;
}

// matmul (matrix.hpp:81-99) on the GPU with the reference's FMA order.
Matrix<float> project(const Matrix<float>& a, const Matrix<float>& b) {
    const auto m = a.rows(), k = a.cols(), n = b.cols();
    Matrix<float> c(m, n);
    if (m == 0 || n == 0) return c;
    DevBuf da(a.data(), a.size() * 4), db(b.data(), b.size() * 4), dc(c.size() * 4);
    check(spl_project(ctx(), da.as<float>(), m, static_cast<std::uint32_t>(k), db.as<float>(),
                      static_cast<std::uint32_t>(n), dc.as<float>(), nullptr));
    finish();
    dc.download(c.data(), c.size() * 4);
    return c;
}
}  // namespace

// oracle_topk (attention_eval.cpp:121-135): exact dense logits + float top-k
// on the GPU (spl_oracle_topk), every query against the shared key matrix.
RetrievalResult oracle_topk(const AttentionInstance& inst, std::uint32_t k) {
    inst.validate();
    if (k == 0) throw DimensionError("oracle_topk: k must be >= 1");
    RetrievalResult res;
    res.method = RetrievalMethod::oracle;
    res.budget = k;
    res.indices = dense_topk(inst.queries.data(), static_cast<std::uint32_t>(inst.num_queries()),
                             inst.keys.data(), static_cast<std::uint32_t>(inst.cache_size()),
                             static_cast<std::uint32_t>(inst.keys.cols()),
                             inst.causal_offsets.data(), inst.scale, k);
    return res;
}

// downproj_topk (attention_eval.cpp:183-206): keys and queries projected by
// the estimator (the reference matmul, GPU), scores = dot of the projections
// (the causal_logits arithmetic with scale 1, exact), float top-k.
RetrievalResult downproj_topk(const AttentionInstance& inst, const DownProjEstimator& est,
                              std::uint32_t k) {
    inst.validate();
    if (k == 0) throw DimensionError("downproj_topk: k must be >= 1");
    if (inst.keys.cols() != est.input_dim())
        throw DimensionError("downproj_topk: estimator dimension mismatch");
    const Matrix<float> kp = project(inst.keys, est.projection);
    const Matrix<float> qp = project(inst.queries, est.projection);
    RetrievalResult res;
    res.method = RetrievalMethod::downproj;
    res.budget = k;
    res.indices = dense_topk(qp.data(), static_cast<std::uint32_t>(qp.rows()), kp.data(),
                             static_cast<std::uint32_t>(kp.rows()), est.reduced_dim(),
                             inst.causal_offsets.data(), 1.0f, k);
    return res;
}

RetrievalResult retrieval_topk(const AttentionInstance& inst, const AnyHasher& hasher,
                               std::uint32_t k) {
    if (const auto* dp = std::get_if<DownProjEstimator>(&hasher)) return downproj_topk(inst, *dp, k);
    return hash_topk(inst, hasher, k);
}

namespace {
// Attention over explicit per-query row lists (own token already inserted):
// one K4 launch in partial-free mode with own-token insertion disabled.
Matrix<float> attend_lists(const AttentionInstance& inst,
                           const std::vector<std::vector<std::uint32_t>>& lists) {
    const auto q = static_cast<std::uint32_t>(inst.num_queries());
    const auto d = static_cast<std::uint32_t>(inst.keys.cols());
    Matrix<float> out(q, d);
    if (q == 0) return out;
    std::size_t kmax = 1;
    for (const auto& l : lists) kmax = std::max(kmax, l.size());
    std::vector<std::uint32_t> idx(static_cast<std::size_t>(q) * kmax, 0), cnt(q);
    for (std::uint32_t r = 0; r < q; ++r) {
        std::copy(lists[r].begin(), lists[r].end(), idx.begin() + static_cast<std::size_t>(r) * kmax);
        cnt[r] = static_cast<std::uint32_t>(lists[r].size());
    }
    // own_row = ~0: attend exactly the given rows (the lists already hold the
    // own token, inserted on the host exactly as the reference does)
    const std::vector<std::uint32_t> no_own(q, 0xFFFFFFFFu);
    DevBuf dq(inst.queries.data(), inst.queries.size() * 4);
    DevBuf dk(inst.keys.data(), inst.keys.size() * 4);
    DevBuf dv(inst.values.data(), inst.values.size() * 4);
    DevBuf di(idx.data(), idx.size() * 4);
    DevBuf dc(cnt.data(), cnt.size() * 4);
    DevBuf downr(no_own.data(), no_own.size() * 4);
    DevBuf dpart(static_cast<std::size_t>(q) * (d + 2) * 4);
    check(spl_sparse_attend_partial(ctx(), dq.as<float>(), dk.as<void>(), dv.as<void>(), SPL_F32, 0, d,
                                    q, di.as<std::uint32_t>(), kmax, dc.as<std::uint32_t>(),
                                    downr.as<std::uint32_t>(), 1, inst.scale, dpart.as<float>(),
                                    nullptr));
    DevBuf dout(out.size() * 4);
    check(spl_attend_combine(ctx(), dpart.as<float>(), 1, q, d, dout.as<float>(), nullptr));
    finish();
    dout.download(out.data(), out.size() * 4);
    return out;
}
}  // namespace

Matrix<float> sparse_attention(const AttentionInstance& inst, const RetrievalResult& result) {
    inst.validate();
    if (result.indices.size() != inst.num_queries())
        throw DimensionError("sparse_attention: result has " + str(result.indices.size()) +
                             " index sets for " + str(inst.num_queries()) + " queries");
    std::vector<std::vector<std::uint32_t>> lists(inst.num_queries());
    for (std::size_t row = 0; row < inst.num_queries(); ++row) {
        const auto& picked = result.indices[row];
        if (picked.empty())
            throw DimensionError("sparse_attention: empty index set for query " + str(row));
        const std::uint32_t valid = inst.causal_offsets[row];
        const std::uint32_t own = valid - 1;
        auto& subset = lists[row];
        subset.assign(picked.begin(), picked.end());
        for (std::uint32_t i : subset)
            if (i >= valid)
                throw DimensionError("sparse_attention: index " + str(i) +
                                     " outside causal range for query " + str(row));
        if (!std::binary_search(subset.begin(), subset.end(), own))
            subset.insert(std::upper_bound(subset.begin(), subset.end(), own), own);
    }
    return attend_lists(inst, lists);
}

Matrix<float> full_attention(const AttentionInstance& inst) {
    inst.validate();
    std::vector<std::vector<std::uint32_t>> lists(inst.num_queries());
    for (std::size_t row = 0; row < inst.num_queries(); ++row) {
        lists[row].resize(inst.causal_offsets[row]);
        for (std::uint32_t i = 0; i < inst.causal_offsets[row]; ++i) lists[row][i] = i;
    }
    return attend_lists(inst, lists);
}

double iou(std::span<const std::uint32_t> a, std::span<const std::uint32_t> b) {
    if (a.empty() && b.empty()) return 1.0;
    std::size_t i = 0, j = 0, both = 0;
    while (i < a.size() && j < b.size()) {
        if (a[i] == b[j]) {
            ++both;
            ++i;
            ++j;
        } else if (a[i] < b[j]) {
            ++i;
        } else {
            ++j;
        }
    }
    return static_cast<double>(both) / static_cast<double>(a.size() + b.size() - both);
}

std::uint32_t budget_from_rate(double rate, std::size_t n) {
    std::uint32_t k = 0;
    if (spl_budget_from_rate(rate, n, &k) != SPL_OK)
        throw DimensionError("budget_from_rate: rate must lie in (0, 1]");
    return k;
}

namespace {
// percentile over ascending values (attention_eval.cpp:276-281): nearest rank
// round(p (size - 1)).
double percentile_sorted(const std::vector<double>& v, double p) {
    if (v.empty()) return 0.0;
    const auto rank = static_cast<std::size_t>(p * static_cast<double>(v.size() - 1) + 0.5);
    return v[std::min(rank, v.size() - 1)];
}
// norm2<float> (matrix.hpp:152-155): sqrt of the float dot, in order.
double norm2f(std::span<const float> a) {
    float acc = 0.0f;
    for (float x : a) acc += x * x;
    return static_cast<double>(std::sqrt(acc));
}
}  // namespace

// evaluate (attention_eval.cpp:285-353): every method at the rate-derived
// budget; per-query IoU against the oracle top-k, output error against full
// attention. Retrieval, attention and the oracle run on the GPU; the
// statistics are host arithmetic over their results.
EvalReport evaluate(const AttentionInstance& inst, std::span<const EvalMethodSpec> methods,
                    double budget_rate) {
    inst.validate();
    const std::uint32_t k = budget_from_rate(budget_rate, inst.cache_size());
    const RetrievalResult oracle = oracle_topk(inst, k);
    const Matrix<float> full = full_attention(inst);
    const std::size_t nq = inst.num_queries();
    std::vector<double> full_norms(nq);
    for (std::size_t r = 0; r < nq; ++r) full_norms[r] = norm2f(full.row(r));
    EvalReport report;
    report.budget = k;
    report.budget_rate = budget_rate;
    for (const EvalMethodSpec& spec : methods) {
        RetrievalResult res;
        if (spec.frozen) {  // every valid row
            res.method = spec.kind;
            res.budget = k;
            res.indices.resize(nq);
            for (std::size_t r = 0; r < nq; ++r) {
                res.indices[r].resize(inst.causal_offsets[r]);
                std::iota(res.indices[r].begin(), res.indices[r].end(), 0u);
            }
        } else if (spec.kind == RetrievalMethod::oracle) {
            res = oracle;
        } else {
            if (!spec.hasher)
                throw DimensionError("evaluate: method \"" + spec.name + "\" needs a hasher");
            res = retrieval_topk(inst, *spec.hasher, k);
        }
        MethodReport mr;
        mr.name = spec.name;
        mr.kind = spec.kind;
        mr.budget = k;
        mr.frozen = spec.frozen;
        mr.per_query_iou.resize(nq);
        const Matrix<float> sparse = sparse_attention(inst, res);
        double iou_sum = 0.0, err_sum = 0.0, err_max = 0.0;
        for (std::size_t r = 0; r < nq; ++r) {
            mr.per_query_iou[r] = iou(res.indices[r], oracle.indices[r]);
            iou_sum += mr.per_query_iou[r];
            double d2 = 0.0;
            for (std::size_t c = 0; c < full.cols(); ++c) {
                const double dl = static_cast<double>(sparse(r, c)) - static_cast<double>(full(r, c));
                d2 += dl * dl;
            }
            const double rel = full_norms[r] > 0.0 ? std::sqrt(d2) / full_norms[r] : std::sqrt(d2);
            err_sum += rel;
            err_max = std::max(err_max, rel);
        }
        mr.mean_iou = iou_sum / static_cast<double>(nq);
        mr.mean_rel_err = err_sum / static_cast<double>(nq);
        mr.max_rel_err = err_max;
        std::vector<double> sorted = mr.per_query_iou;
        std::sort(sorted.begin(), sorted.end());
        mr.p10_iou = percentile_sorted(sorted, 0.10);
        mr.p50_iou = percentile_sorted(sorted, 0.50);
        mr.p90_iou = percentile_sorted(sorted, 0.90);
        report.methods.push_back(std::move(mr));
    }
    return report;
}

// format_eval_report (attention_eval.cpp:355-373): provenance lines, budget,
// one record per method — same fields and number formats.
std::string format_eval_report(const EvalReport& report, std::span<const std::string> header_lines) {
    std::string out;
    for (const std::string& h : header_lines) out += "# " + h + "\n";
    char buf[320];
    std::snprintf(buf, sizeof(buf), "budget %u\n", report.budget);
    out += buf;
    {
        std::ostringstream os;
        os << report.budget_rate;  // default stream formatting, as the reference prints it
        out += "budget_rate " + os.str() + "\n";
    }
    for (const MethodReport& m : report.methods) {
        std::snprintf(buf, sizeof(buf),
                      "method %s kind=%s budget=%u frozen=%d mean_iou=%.6f p10=%.6f p50=%.6f "
                      "p90=%.6f mean_rel_err=%.6e max_rel_err=%.6e\n",
                      m.name.c_str(), retrieval_method_name(m.kind), m.budget, m.frozen ? 1 : 0,
                      m.mean_iou, m.p10_iou, m.p50_iou, m.p90_iou, m.mean_rel_err, m.max_rel_err);
        out += buf;
    }
    return out;
}

// eval_report_csv (attention_eval.cpp:375-391): per-query IoU, one column per method.
std::string eval_report_csv(const EvalReport& report) {
    std::string out = "query";
    for (const MethodReport& m : report.methods) out += "," + m.name;
    out += "\n";
    if (report.methods.empty()) return out;
    char buf[32];
    for (std::size_t r = 0; r < report.methods.front().per_query_iou.size(); ++r) {
        out += std::to_string(r);
        for (const MethodReport& m : report.methods) {
            std::snprintf(buf, sizeof(buf), ",%.6f", m.per_query_iou[r]);
            out += buf;
        }
        out += "\n";
    }
    return out;
}

// ------------------------------------------------------------ training (§8 f4)
void RankingLossConfig::validate(std::size_t n_keys) const {  // ranking_loss.cpp:13-28
    if (beta <= 0.0) throw DimensionError("ranking loss: beta must be positive");
    if (!(maskout > 0.0 && maskout < 1.0)) throw DimensionError("ranking loss: maskout must lie in (0, 1)");
    const auto k = static_cast<std::uint32_t>(static_cast<double>(n_keys) * (1.0 - maskout));
    if (k == 0) throw DimensionError("ranking loss: top count floored to zero for n=" + str(n_keys));
    if (max_top && *max_top == 0) throw DimensionError("ranking loss: max_top must be >= 1");
    if (max_oth && *max_oth == 0) throw DimensionError("ranking loss: max_oth must be >= 1");
    if (query_subsample && *query_subsample == 0)
        throw DimensionError("ranking loss: query_subsample must be >= 1");
}

namespace {
spl_train_config to_c(const TrainConfig& c) {
    spl_train_config t{};
    t.num_iters = c.num_iters;
    t.warmup_iters = c.warmup_iters;
    t.batch = c.batch;
    t.holdout_queries = c.holdout_queries;
    t.seed = c.seed;
    t.max_lr = c.max_lr;
    t.min_lr = c.min_lr;
    t.adam_beta1 = c.adam_beta1;
    t.adam_beta2 = c.adam_beta2;
    t.adam_eps = c.adam_eps;
    t.weight_decay = c.weight_decay;
    t.grad_clip = c.grad_clip;
    t.soft_gamma = c.soft_gamma;
    t.holdout_budget_rate = c.holdout_budget_rate;
    return t;
}
}  // namespace

// SPLQ dumps (synthkv.cpp:104-142)
void write_dump(const std::string& path, const Matrix<float>& queries, const Matrix<float>& keys) {
    if (queries.cols() != keys.cols()) throw DimensionError("write_dump: query and key dimensions differ");
    auto finite = [](const Matrix<float>& m) {
        for (std::size_t i = 0; i < m.size(); ++i)
            if (!std::isfinite(m.data()[i])) return false;
        return true;
    };
    if (!finite(queries) || !finite(keys)) throw NumericError("write_dump: tensors contain non-finite values");
    auto os = open_out(path);
    os.write("SPLQ", 4);
    write_u32(os, 1);
    write_u32(os, static_cast<std::uint32_t>(queries.rows()));
    write_u32(os, static_cast<std::uint32_t>(keys.rows()));
    write_u32(os, static_cast<std::uint32_t>(queries.cols()));
    write_words(os, queries.data(), queries.size());
    write_words(os, keys.data(), keys.size());
    if (!os) throw IoError("write failed: " + path);
}

QkDump read_dump(const std::string& path) {
    Reader r(path);
    r.magic("SPLQ");
    const std::uint32_t version = r.u32("version");
    if (version != 1) throw FormatError(path + ": unsupported SPLQ version " + str(version));
    const std::uint32_t nq = r.u32("n_queries");
    const std::uint32_t nk = r.u32("n_keys");
    const std::uint32_t d = r.u32("d");
    QkDump dump{Matrix<float>(nq, d), Matrix<float>(nk, d)};
    r.words(dump.queries.data(), dump.queries.size(), "query block");
    r.words(dump.keys.data(), dump.keys.size(), "key block");
    for (const Matrix<float>* m : {&dump.queries, &dump.keys})
        for (std::size_t i = 0; i < m->size(); ++i)
            if (!std::isfinite(m->data()[i])) throw FormatError(path + ": payload contains non-finite values");
    return dump;
}

TrainDataset dataset_from_dump(QkDump dump) {
    TrainDataset data;
    data.sequences.push_back(QkSequence{std::move(dump.queries), std::move(dump.keys)});
    return data;
}

void TrainConfig::validate() const {  // trainer.cpp:19-33
    if (max_lr < 0.0 || min_lr < 0.0 || min_lr > max_lr)
        throw DimensionError("TrainConfig: need 0 <= min_lr <= max_lr");
    if (!(adam_beta1 >= 0.0 && adam_beta1 < 1.0 && adam_beta2 >= 0.0 && adam_beta2 < 1.0))
        throw DimensionError("TrainConfig: adam betas must lie in [0, 1)");
    if (adam_eps <= 0.0) throw DimensionError("TrainConfig: adam_eps must be positive");
    if (weight_decay < 0.0) throw DimensionError("TrainConfig: weight_decay must be >= 0");
    if (batch < 1) throw DimensionError("TrainConfig: batch must be >= 1");
    if (soft_gamma <= 0.0) throw DimensionError("TrainConfig: soft_gamma must be positive");
    if (!(holdout_budget_rate > 0.0 && holdout_budget_rate <= 1.0))
        throw DimensionError("TrainConfig: holdout_budget_rate must lie in (0, 1]");
}

double lr_at(std::uint32_t iter, const TrainConfig& cfg) {
    const spl_train_config c = to_c(cfg);
    return spl_train_lr_at(iter, &c);
}

std::string format_train_report(const TrainReport& report,
                                std::span<const std::string> header_lines) {  // trainer.cpp:152-175
    std::string out;
    for (const std::string& line : header_lines) out += "# " + line + "\n";
    out += "# columns: iter loss violation_rate lr\n";
    char buf[160];
    for (const IterRecord& rec : report.records) {
        std::snprintf(buf, sizeof(buf), "%u %.9g %.9g %.9g", rec.iter, rec.loss, rec.violation_rate,
                      rec.lr);
        out += buf;
        out += "\n";
    }
    std::snprintf(buf, sizeof(buf), "# final_holdout_iou %.6f", report.final_holdout_iou);
    out += buf;
    out += "\n# skipped_steps " + std::to_string(report.skipped_steps) + "\n";
    return out;
}

TrainReport train_hasher(AnyHasher& hasher, const TrainDataset& dataset,
                         const RankingLossConfig& loss_cfg, const TrainConfig& cfg,
                         TrainLoss loss_kind) {
    const auto t0 = std::chrono::steady_clock::now();
    cfg.validate();
    if (dataset.sequences.empty()) throw DimensionError("train_hasher: dataset is empty");
    std::vector<float> qs, ks;
    std::vector<std::uint32_t> lens;
    std::uint32_t d = 0;
    for (const QkSequence& seq : dataset.sequences) {
        if (seq.queries.rows() != seq.keys.rows())
            throw DimensionError("train_hasher: queries and keys must be causally aligned");
        if (seq.queries.rows() < 2)
            throw DimensionError("train_hasher: sequences need at least two positions");
        d = static_cast<std::uint32_t>(seq.queries.cols());
        qs.insert(qs.end(), seq.queries.data(), seq.queries.data() + seq.queries.size());
        ks.insert(ks.end(), seq.keys.data(), seq.keys.data() + seq.keys.size());
        lens.push_back(static_cast<std::uint32_t>(seq.queries.rows()));
    }
    spl_rank_config rc{loss_cfg.beta, loss_cfg.alpha, loss_cfg.maskout,
                       loss_cfg.max_top ? static_cast<std::int64_t>(*loss_cfg.max_top) : -1,
                       loss_cfg.max_oth ? static_cast<std::int64_t>(*loss_cfg.max_oth) : -1,
                       loss_cfg.query_subsample ? static_cast<std::int64_t>(*loss_cfg.query_subsample) : -1};
    const spl_train_config tc = to_c(cfg);
    std::vector<double> rec(static_cast<std::size_t>(cfg.num_iters) * 3 + 3);
    double iou = 0.0;
    std::uint32_t skipped = 0;
    auto dim_check = [&](std::uint32_t in_dim) {
        if (in_dim != d)
            throw DimensionError("train_hasher: data dimension " + std::to_string(d) +
                                 " does not match hasher dimension " + std::to_string(in_dim));
    };
    const int lk = loss_kind == TrainLoss::reconstruction ? SPL_TRAIN_LOSS_RECONSTRUCTION
                                                          : SPL_TRAIN_LOSS_RANKING;
    spl_status st = SPL_OK;
    if (auto* m = std::get_if<MlpHasher>(&hasher)) {
        dim_check(m->input_dim());
        st = spl_train_hasher(ctx(), SPL_HASHER_MLP, m->input_dim(), m->hidden_dim(), m->code_bits(),
                              m->gamma, m->w1.data(), m->b1.data(), m->w2.data(),
                              static_cast<std::uint32_t>(lens.size()), qs.data(), ks.data(),
                              lens.data(), &rc, &tc, lk, rec.data(), &iou, &skipped, nullptr);
    } else if (auto* l = std::get_if<LinearHasher>(&hasher)) {
        dim_check(l->input_dim());
        st = spl_train_hasher(ctx(), SPL_HASHER_LINEAR, l->input_dim(), 0, l->code_bits(), 0.0f,
                              l->projection.data(), nullptr, nullptr,
                              static_cast<std::uint32_t>(lens.size()), qs.data(), ks.data(),
                              lens.data(), &rc, &tc, lk, rec.data(), &iou, &skipped, nullptr);
    } else {
        auto& e = std::get<DownProjEstimator>(hasher);
        dim_check(e.input_dim());
        st = spl_train_hasher(ctx(), SPL_HASHER_DOWNPROJ, e.input_dim(), 0, e.reduced_dim(), 0.0f,
                              e.projection.data(), nullptr, nullptr,
                              static_cast<std::uint32_t>(lens.size()), qs.data(), ks.data(),
                              lens.data(), &rc, &tc, lk, rec.data(), &iou, &skipped, nullptr);
    }
    check(st);
    TrainReport report;
    report.records.reserve(cfg.num_iters);
    for (std::uint32_t it = 0; it < cfg.num_iters; ++it)
        report.records.push_back(IterRecord{it, rec[3 * static_cast<std::size_t>(it)],
                                            rec[3 * static_cast<std::size_t>(it) + 1],
                                            rec[3 * static_cast<std::size_t>(it) + 2]});
    report.final_holdout_iou = iou;
    report.skipped_steps = skipped;
    report.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return report;
}

}  // namespace spotlight
