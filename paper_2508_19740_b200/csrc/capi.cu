// extern "C" entry points of include/spl_c.h: argument validation with the
// reference's error wording, context / workspace management, dispatch to the
// sm_100a kernels. No CPU compute path exists: every compute entry point
// launches a kernel or fails.
#include <cuda.h>  // driver types only (entry points fetched through cudart)
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <vector>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "spl_launch.cuh"
#include "spl_tc.cuh"


using namespace spl;

namespace spl {
bool pdl_enabled() {
    // off by default: measured on B200 it cost more than it hid (config-3
    // retrieval 59.2 -> 61.9 us, config-2 decode step 58.1 -> 59.5 us;
    // config-4 step 689 -> 684 us). SPL_PDL=1 turns it on.
    static const bool on = [] {
        const char* e = getenv("SPL_PDL");
        return e && *e == '1';
    }();
    return on;
}
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       void** args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, fn, args);
}
}  // namespace spl

namespace {
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
// NVTX range around each compute entry point (no cost without a profiler)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
constexpr float kLog2e = 1.4426950408889634f;


spl_status check_L(spl_ctx* ctx, const char* who, uint32_t L) {
    if (L == 0 || L % 32 != 0)
        return fail(ctx, SPL_E_DIMENSION,
                    std::string(who) + ": column count " + std::to_string(L) +
                        " must be a positive multiple of 32");
    if (L > (1u << 15))
        return fail(ctx, SPL_E_DIMENSION,
                    std::string("CodeMatrix: length_bits ") + std::to_string(L) +
                        " exceeds the 32768-bit limit");
    return SPL_OK;
}
}  // namespace

extern "C" {

const char* spl_version(void) { return "spotlight-b200 0.1 (sm_100a)"; }

namespace {
// SMs this context may actually use. A green context (or any context created
// on an SM partition) reports its share through cuCtxGetDevResource; MPS
// clients are capped by CUDA_MPS_ACTIVE_THREAD_PERCENTAGE. Either way the
// fused K3 kernel's CTAs may not all be resident at once, so such contexts
// launch it cooperatively (the driver then guarantees co-residency or refuses,
// and the retrieval falls back to the two-pass kernels). Returns the usable
// SM count; *limited is set when it is below the device's.
int usable_sms(int device_sms, bool* limited) {
    *limited = false;
    int sms = device_sms;
    using GetCurrent = CUresult (*)(CUcontext*);
    using GetRes = CUresult (*)(CUcontext, CUdevResource*, CUdevResourceType);
    void* f_cur = nullptr;
    void* f_res = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &f_cur, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuCtxGetDevResource", &f_res, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && f_cur && f_res) {
        CUcontext cu = nullptr;
        CUdevResource res;
        memset(&res, 0, sizeof(res));
        if (reinterpret_cast<GetCurrent>(f_cur)(&cu) == CUDA_SUCCESS && cu &&
            reinterpret_cast<GetRes>(f_res)(cu, &res, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS &&
            res.sm.smCount > 0 && (int)res.sm.smCount < sms)
            sms = (int)res.sm.smCount;
    }
    cudaGetLastError();
    if (const char* e = getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE")) {
        const double pct = atof(e);
        if (pct > 0.0 && pct < 100.0) sms = std::max(1, std::min(sms, (int)(device_sms * pct / 100.0)));
    }
    *limited = sms < device_sms;
    return sms;
}
}  // namespace

spl_status spl_ctx_create(int device, spl_ctx** out) {
    if (!out) return SPL_E_STATE;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return SPL_E_CUDA;
    }
    if (device < 0 || device >= n) return SPL_E_CUDA;
    if (cudaSetDevice(device) != cudaSuccess) return SPL_E_CUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SPL_E_CUDA;
    if (prop.major != 10) {
        // sm_100a cubins only: fail loudly on anything that is not Blackwell.
        return SPL_E_CUDA;
    }
    spl_ctx* c = new spl_ctx;
    c->device = device;
    bool limited = false;
    c->num_sms = usable_sms(prop.multiProcessorCount, &limited);
    c->k3_coop = limited;
    if (cudaMalloc(&c->dev_err, sizeof(uint32_t)) != cudaSuccess ||
        cudaMemset(c->dev_err, 0, sizeof(uint32_t)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        delete c;
        return SPL_E_CUDA;
    }
    *out = c;
    return SPL_OK;
}

void spl_ctx_destroy(spl_ctx* ctx) {
    if (!ctx) return;
    cudaDeviceSynchronize();
    cudaFree(ctx->dev_err);
    cudaFree(ctx->k3_ws);
    cudaFree(ctx->k3_state);
    cudaFree(ctx->att_ws);
    cudaFree(ctx->att_counters);
    cudaFree(ctx->scratch);
    cudaFree(ctx->dense_ws);
    delete ctx;
}

const char* spl_last_error(const spl_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

uint64_t spl_launch_count(const spl_ctx* ctx) { return ctx ? ctx->launches : 0; }

size_t spl_launch_log(spl_ctx* ctx, char* buf, size_t len) {
    if (!ctx) return 0;
    const size_t n = ctx->launch_log.size();
    if (buf && len) {
        const size_t m = n < len - 1 ? n : len - 1;
        memcpy(buf, ctx->launch_log.data(), m);
        buf[m] = '\0';
    }
    ctx->launch_log.clear();
    return n;
}

// Size every workspace a call on up to (P, n_max, L, k, d) can touch, on
// stream s (spl_reserve: the legacy stream), so the calls themselves never
// allocate: required before CUDA-graph capture, and before the first step
// of a peer group whose kernels wait for each other inside.
spl_status reserve_impl(spl_ctx* ctx, uint32_t P, uint64_t n_max, uint32_t L, uint32_t k,
                        uint32_t d, cudaStream_t s) {
    // Run each path once on a dummy problem set sized like the real one is
    // not possible without data; size the buffers from the same formulas.
    const size_t score_bytes = L <= 256 ? 1 : 2;
    const size_t n_pad = (n_max + 63) / 64 * 64;
    const size_t G = (size_t)ctx->num_sms * 8 + 1;
    const size_t sc = ((size_t)P * n_pad * score_bytes + 255) / 256 * 256;
    const size_t rec = ((G + P) * (L + 2) * 4 + 255) / 256 * 256;
    const size_t plans = ((G + P) * 16 + 255) / 256 * 256;
    spl_status st = ensure_buffer(ctx, &ctx->k3_ws, &ctx->k3_ws_bytes, sc + rec + plans, false,
                                  s, "spl_reserve");
    if (st) return st;
    size_t have = ctx->k3_state_words * 4;
    st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->k3_state), &have,
                       (2 + (size_t)P * (1 + (L + 2) + 4)) * 4, true, s, "spl_reserve");
    if (st) return st;
    ctx->k3_state_words = have / 4;
    // decode-step query codes
    st = ensure_buffer(ctx, &ctx->scratch, &ctx->scratch_bytes, (size_t)P * (L / 32) * 4 + 4 * (size_t)P,
                       false, s, "spl_reserve");
    if (st) return st;
    if (d > 0) {
        if ((st = sparse_attend_reserve(ctx, P, k, d, s))) return st;
        // the fused decode step's per-segment partials [(G + P)][d + 2]
        st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_ws), &ctx->att_ws_bytes,
                           (G + P) * ((size_t)(d > 128 ? d : 128) + 2) * 4, false, s, "spl_reserve");
        if (st) return st;
        // the sharded step's partials [P][d + 2]
        st = ensure_buffer(ctx, &ctx->dense_ws, &ctx->dense_ws_bytes, (size_t)P * (d + 2) * 4, false, s,
                           "spl_reserve");
        if (st) return st;
    }
    return SPL_OK;
}

spl_status spl_reserve(spl_ctx* ctx, uint32_t P, uint64_t n_max, uint32_t L, uint32_t k,
                       uint32_t d) {
    if (!ctx) return SPL_E_STATE;
    return reserve_impl(ctx, P, n_max, L, k, d, 0);
}

spl_status spl_check_device_error(spl_ctx* ctx, void* stream) {
    if (!ctx) return SPL_E_STATE;
    uint32_t flags = 0;
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(&flags, ctx->dev_err, 4, cudaMemcpyDeviceToHost, S(stream)));
    SPL_CUDA_TRY(ctx, cudaStreamSynchronize(S(stream)));
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(ctx->dev_err, 0, 4, S(stream)));
    SPL_CUDA_TRY(ctx, cudaStreamSynchronize(S(stream)));
    if (flags & SPL_DEV_ERR_NUMERIC)
        return fail(ctx, SPL_E_NUMERIC, "mlp input contains non-finite values");
    if (flags & SPL_DEV_ERR_DIMENSION)
        return fail(ctx, SPL_E_DIMENSION,
                    "decode: causal offset / append slot outside the cache (n_valid == 0 or >= capacity)");
    if (flags & SPL_DEV_ERR_STALL)
        return fail(ctx, SPL_E_CUDA,
                    "hamming_topk: fused kernel CTAs were not co-resident (watchdog); "
                    "set SPL_K3_COOP=1 or SPL_K3_PATH=twopass");
    return SPL_OK;
}

spl_status spl_device_alloc(spl_ctx* ctx, size_t bytes, void** out) {
    if (!out) return SPL_E_STATE;
    SPL_CUDA_TRY(ctx, cudaMalloc(out, bytes ? bytes : 1));
    return SPL_OK;
}
spl_status spl_device_free(spl_ctx* ctx, void* p) {
    SPL_CUDA_TRY(ctx, cudaFree(p));
    return SPL_OK;
}
spl_status spl_memcpy(spl_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream) {
    if (bytes == 0) return SPL_OK;
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, S(stream)));
    return SPL_OK;
}
spl_status spl_memset(spl_ctx* ctx, void* dst, int value, size_t bytes, void* stream) {
    if (bytes == 0) return SPL_OK;
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(dst, value, bytes, S(stream)));
    return SPL_OK;
}
spl_status spl_stream_synchronize(spl_ctx* ctx, void* stream) {
    SPL_CUDA_TRY(ctx, cudaStreamSynchronize(S(stream)));
    return SPL_OK;
}

// ------------------------------------------------------------ bitcodes
spl_status spl_pack_bits(spl_ctx* ctx, const uint8_t* bits, uint64_t n, uint32_t L,
                         uint32_t* codes, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (L == 0 || L % 32 != 0)
        return fail(ctx, SPL_E_DIMENSION,
                    "pack_bits: column count " + std::to_string(L) +
                        " must be a positive multiple of 32");
    if (spl_status st = check_L(ctx, "pack_bits", L)) return st;
    return pack_bits_launch(ctx, bits, n, L, codes, S(stream));
}

spl_status spl_unpack_bits(spl_ctx* ctx, const uint32_t* codes, uint64_t n, uint32_t L,
                           uint8_t* bits, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (spl_status st = check_L(ctx, "unpack_bits", L)) return st;
    return unpack_bits_launch(ctx, codes, n, L, bits, S(stream));
}

spl_status spl_nxor_scores(spl_ctx* ctx, const uint32_t* codes, uint64_t problem_stride_rows,
                           uint32_t L, const uint32_t* qcodes, uint32_t P,
                           const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                           int32_t* scores, uint64_t scores_stride, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (spl_status st = check_L(ctx, "nxor_scores", L)) return st;
    if (nvalid_div == 0) return fail(ctx, SPL_E_DIMENSION, "nxor_scores: nvalid_div == 0");
    return nxor_scores_launch(ctx, codes, problem_stride_rows, L, qcodes, P, n_valid, nvalid_div,
                              n_max, scores, scores_stride, S(stream));
}

spl_status spl_top_k(spl_ctx* ctx, const void* scores, int dtype, uint32_t P, uint64_t n,
                     uint64_t scores_stride, uint32_t k, uint32_t* idx, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (k == 0 || k > n)
        return fail(ctx, SPL_E_DIMENSION,
                    "top_k_indices: k=" + std::to_string(k) + " out of range for n=" +
                        std::to_string(n));
    return top_k_launch(ctx, scores, dtype, P, n, scores_stride, k, idx, S(stream));
}

// ------------------------------------------------ peer group (fused sharding)
spl_status spl_peer_create(spl_ctx* ctx, uint32_t R, uint32_t rank, uint32_t P_max,
                           uint32_t L_max, spl_peer** out) {
    if (!ctx || !out) return SPL_E_STATE;
    *out = nullptr;
    if (R == 0 || rank >= R || P_max == 0 || L_max == 0 || L_max % 32 != 0 || L_max > (1u << 15))
        return fail(ctx, SPL_E_DIMENSION, "peer_create: need 0 <= rank < R, P_max >= 1, L_max % 32 == 0");
    // the group's kernels wait for each other inside: load every kernel a
    // sharded call can launch now, not lazily in the middle of a step
    encode_preload();
    attend_preload();
    k3_preload();
    auto* pe = new spl_peer;
    pe->R = R;
    pe->rank = rank;
    pe->Pmax = P_max;
    pe->Lmax = L_max;
    pe->device = ctx->device;
    pe->bytes = peer_area_words(R, P_max, L_max) * 4;
    cudaError_t e = cudaMalloc(&pe->buf, pe->bytes);
    if (e == cudaSuccess) e = cudaMemset(pe->buf, 0, pe->bytes);
    if (e == cudaSuccess) e = cudaMalloc(&pe->d_table, sizeof(uint32_t*) * R);
    if (e == cudaSuccess) e = cudaMalloc(&pe->d_epoch, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(pe->d_epoch, 0, sizeof(uint32_t));
    // legacy-stream memsets are not ordered before non-blocking streams:
    // complete them before any kernel can touch the exchange area
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(pe->buf);
        delete pe;
        return cuda_fail(ctx, e, "peer_create");
    }
    *out = pe;
    return SPL_OK;
}

spl_status spl_peer_ipc_handle(spl_ctx* ctx, const spl_peer* peer, void* handle) {
    if (!ctx || !peer || !handle) return SPL_E_STATE;
    cudaIpcMemHandle_t h;
    SPL_CUDA_TRY(ctx, cudaIpcGetMemHandle(&h, peer->buf));
    std::memcpy(handle, &h, sizeof(h));
    return SPL_OK;
}

spl_status spl_peer_open(spl_ctx* ctx, spl_peer* peer, const void* handles) {
    if (!ctx || !peer || !handles) return SPL_E_STATE;
    std::vector<uint32_t*> table(peer->R, nullptr);
    for (uint32_t r = 0; r < peer->R; ++r) {
        if (r == peer->rank) {
            table[r] = peer->buf;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof(h), sizeof(h));
        void* ptr = nullptr;
        SPL_CUDA_TRY(ctx, cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        peer->opened.push_back(ptr);
        table[r] = static_cast<uint32_t*>(ptr);
    }
    SPL_CUDA_TRY(ctx, cudaMemcpy(peer->d_table, table.data(), sizeof(uint32_t*) * peer->R,
                                 cudaMemcpyHostToDevice));
    peer->connected = true;
    return SPL_OK;
}

spl_status spl_peer_connect_local(spl_ctx* ctx, spl_peer* const* peers, uint32_t R) {
    if (!ctx || !peers || R == 0) return SPL_E_STATE;
    std::vector<uint32_t*> table(R);
    for (uint32_t r = 0; r < R; ++r) {
        if (!peers[r] || peers[r]->R != R || peers[r]->rank != r)
            return fail(ctx, SPL_E_DIMENSION, "peer_connect_local: peers must be ranks 0..R-1 of one group");
        table[r] = peers[r]->buf;
    }
    for (uint32_t r = 0; r < R; ++r) {
        SPL_CUDA_TRY(ctx, cudaMemcpy(peers[r]->d_table, table.data(), sizeof(uint32_t*) * R,
                                     cudaMemcpyHostToDevice));
        peers[r]->connected = true;
    }
    return SPL_OK;
}

void spl_peer_destroy(spl_peer* peer) {
    if (!peer) return;
    cudaDeviceSynchronize();
    for (void* p : peer->opened) cudaIpcCloseMemHandle(p);
    cudaFree(peer->d_table);
    cudaFree(peer->d_epoch);
    cudaFree(peer->buf);
    delete peer;
}

spl_status spl_hamming_topk_sharded(spl_ctx* ctx, spl_peer* peer, const uint32_t* codes,
                                    uint64_t problem_stride_rows, uint32_t L,
                                    const uint32_t* qcodes, uint32_t P, const uint32_t* n_valid,
                                    uint32_t nvalid_div, uint64_t n_max, uint32_t k,
                                    uint32_t* idx, uint32_t* cnt, uint32_t* out_offset,
                                    void* stream) {
    NvtxRange nvtx_("spl_hamming_topk_sharded");
    return hamming_topk_sharded_impl(ctx, peer, codes, problem_stride_rows, L, qcodes, P, n_valid,
                                     nvalid_div, n_max, k, idx, cnt, out_offset, S(stream));
}

// ------------------------------------------------ dense retrieval (§8 f2)
spl_status spl_oracle_topk(spl_ctx* ctx, const float* q, const void* keys, int kv_dtype,
                           uint64_t cap, uint32_t d, uint32_t P, const uint32_t* n_valid,
                           uint32_t nvalid_div, uint64_t n_max, float scale, uint32_t k,
                           uint32_t* idx, uint32_t* cnt, float* logits, void* stream) {
    NvtxRange nvtx_("spl_oracle_topk");
    if (!ctx) return SPL_E_STATE;
    if (k == 0) return fail(ctx, SPL_E_DIMENSION, "oracle_topk: k must be >= 1");
    if (kv_dtype != SPL_F32 && kv_dtype != SPL_BF16)
        return fail(ctx, SPL_E_DIMENSION, "oracle_topk: unknown key dtype");
    if (nvalid_div == 0) return fail(ctx, SPL_E_DIMENSION, "oracle_topk: nvalid_div == 0");
    if (P == 0 || n_max == 0) return SPL_OK;
    if (!q || !keys || !n_valid || !idx || !cnt)
        return fail(ctx, SPL_E_STATE, "oracle_topk: null device pointer");
    if (!logits) {
        spl_status st = ensure_buffer(ctx, &ctx->dense_ws, &ctx->dense_ws_bytes,
                                      (size_t)P * n_max * sizeof(float), false, S(stream),
                                      "oracle_topk");
        if (st) return st;
        logits = static_cast<float*>(ctx->dense_ws);
    }
    spl_status st = causal_logits_launch(ctx, q, keys, kv_dtype, cap, d, P, n_valid, nvalid_div,
                                         n_max, scale, logits, S(stream));
    if (st) return st;
    return top_k_launch(ctx, logits, 1, P, n_max, n_max, k, idx, S(stream), n_valid, nvalid_div,
                        cnt);
}

spl_status spl_project(spl_ctx* ctx, const float* a, uint64_t m, uint32_t k, const float* b,
                       uint32_t n, float* c, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (k == 0) return fail(ctx, SPL_E_DIMENSION, "matmul: inner dimension must be >= 1");
    if (m && n && (!a || !b || !c)) return fail(ctx, SPL_E_STATE, "matmul: null device pointer");
    return project_launch(ctx, a, m, k, b, n, c, S(stream));
}

spl_status spl_iou(spl_ctx* ctx, const uint32_t* a, const uint32_t* cnt_a, uint64_t a_stride,
                   const uint32_t* b, const uint32_t* cnt_b, uint64_t b_stride, uint32_t P,
                   double* out, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (P == 0) return SPL_OK;
    if (!a || !cnt_a || !b || !cnt_b || !out) return fail(ctx, SPL_E_STATE, "iou: null device pointer");
    return iou_launch(ctx, a, cnt_a, a_stride, b, cnt_b, b_stride, P, out, S(stream));
}

// ------------------------------------------------------------ K3
spl_status spl_hamming_topk(spl_ctx* ctx, const uint32_t* codes, uint64_t problem_stride_rows,
                            uint32_t L, const uint32_t* qcodes, uint32_t P,
                            const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                            uint32_t k, uint32_t* idx, uint32_t* cnt, void* stream) {
    NvtxRange nvtx_("spl_hamming_topk");
    return hamming_topk_impl(ctx, codes, problem_stride_rows, L, qcodes, P, n_valid, nvalid_div,
                             n_max, k, idx, cnt, S(stream));
}

spl_status spl_shard_histogram(spl_ctx* ctx, const uint32_t* codes,
                               uint64_t problem_stride_rows, uint32_t L,
                               const uint32_t* qcodes, uint32_t P, const uint32_t* n_valid,
                               uint32_t nvalid_div, uint64_t n_max, uint32_t* hist,
                               void* stream) {
    NvtxRange nvtx_("spl_shard_histogram");
    return shard_histogram_impl(ctx, codes, problem_stride_rows, L, qcodes, P, n_valid,
                                nvalid_div, n_max, hist, S(stream));
}

spl_status spl_shard_select(spl_ctx* ctx, const uint32_t* all_hist, uint32_t R, uint32_t rank,
                            uint32_t L, uint32_t P, const uint32_t* n_valid,
                            uint32_t nvalid_div, uint64_t n_max, uint32_t k, uint32_t* idx,
                            uint32_t* cnt, uint32_t* out_offset, void* stream) {
    NvtxRange nvtx_("spl_shard_select");
    return shard_select_impl(ctx, all_hist, R, rank, L, P, n_valid, nvalid_div, n_max, k, idx,
                             cnt, out_offset, S(stream));
}

// ------------------------------------------------------------ encoders
spl_status spl_hasher_create(spl_ctx* ctx, int kind, uint32_t H, uint32_t d, uint32_t h,
                             uint32_t L, const float* w1, const float* b1, const float* w2,
                             spl_hasher** out) {
    if (!ctx || !out) return SPL_E_STATE;
    *out = nullptr;
    if (kind != SPL_HASHER_MLP && kind != SPL_HASHER_LINEAR)
        return fail(ctx, SPL_E_DIMENSION, "hasher: unknown kind");
    if (H == 0 || d == 0 || (kind == SPL_HASHER_MLP && h == 0))
        return fail(ctx, SPL_E_DIMENSION, "mlp_gaussian_init: dimensions must be >= 1");
    if (spl_status st = check_L(ctx, "pack_bits", L)) return st;
    if (!w1 || (kind == SPL_HASHER_MLP && (!b1 || !w2)))
        return fail(ctx, SPL_E_STATE, "hasher: null weight pointer");
    const size_t n1 = (size_t)H * d * (kind == SPL_HASHER_MLP ? h : L);
    const size_t nb = kind == SPL_HASHER_MLP ? (size_t)H * h : 0;
    const size_t n2 = kind == SPL_HASHER_MLP ? (size_t)H * h * L : 0;
    // require_finite (hashers.cpp:14-17, :90-95) on a host copy
    std::vector<float> h1(n1), hb(nb), h2(n2);
    SPL_CUDA_TRY(ctx, cudaMemcpy(h1.data(), w1, n1 * 4, cudaMemcpyDefault));
    if (nb) SPL_CUDA_TRY(ctx, cudaMemcpy(hb.data(), b1, nb * 4, cudaMemcpyDefault));
    if (n2) SPL_CUDA_TRY(ctx, cudaMemcpy(h2.data(), w2, n2 * 4, cudaMemcpyDefault));
    for (float v : h1)
        if (!std::isfinite(v)) return fail(ctx, SPL_E_NUMERIC, "mlp w1 contains non-finite values");
    for (float v : h2)
        if (!std::isfinite(v)) return fail(ctx, SPL_E_NUMERIC, "mlp w2 contains non-finite values");
    for (float v : hb)
        if (!std::isfinite(v)) return fail(ctx, SPL_E_NUMERIC, "mlp b1 is non-finite");
    spl_hasher* hs = new spl_hasher;
    hs->kind = kind;
    hs->H = H;
    hs->d = d;
    hs->h = kind == SPL_HASHER_MLP ? h : 0;
    hs->L = L;
    auto up = [&](float** dst, const std::vector<float>& src) -> bool {
        if (src.empty()) return true;
        if (cudaMalloc(dst, src.size() * 4) != cudaSuccess) return false;
        return cudaMemcpy(*dst, src.data(), src.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    // layer-2 (linear: projection) columns permuted [p][c*W + w] -> [p][w*32 + c]
    // so the encoder's warp on word w reads 32 consecutive floats per step
    const std::vector<float>& src2 = kind == SPL_HASHER_MLP ? h2 : h1;
    const uint32_t rows2 = kind == SPL_HASHER_MLP ? h : d, W = L / 32;
    std::vector<float> hp(src2.size());
    for (uint32_t hd = 0; hd < H; ++hd)
        for (uint32_t p = 0; p < rows2; ++p)
            for (uint32_t c = 0; c < 32; ++c)
                for (uint32_t w = 0; w < W; ++w)
                    hp[((size_t)hd * rows2 + p) * L + w * 32 + c] =
                        src2[((size_t)hd * rows2 + p) * L + c * W + w];
    // cluster-encoder layouts (encode_exact.cu, fma_chain2): W1 column
    // quarters [H][4][h/4][d] and layer 2 word-major [H][W][32][rows2], both
    // with one row per output (lane-major), so each CTA's block is contiguous
    // and a lane's weights are consecutive; chunk c (4 floats) of the row of
    // output j is stored at chunk slot (c + j mod 32) mod (row / 4), which
    // makes the per-lane 16-byte loads bank-conflict free.
    auto rot = [](uint32_t p, uint32_t lane, uint32_t n) {
        const uint32_t nc = n / 4;
        return ((p / 4 + lane) % nc) * 4 + p % 4;
    };
    std::vector<float> hs1, hw2;
    const bool cl_ok = d % 4 == 0 && rows2 % 4 == 0;
    if (kind == SPL_HASHER_MLP && h % 4 == 0 && cl_ok) {
        const uint32_t q = h / 4;
        hs1.resize(h1.size());
        for (uint32_t hd = 0; hd < H; ++hd)
            for (uint32_t r = 0; r < 4; ++r)
                for (uint32_t jj = 0; jj < q; ++jj)
                    for (uint32_t p = 0; p < d; ++p)
                        hs1[(((size_t)hd * 4 + r) * q + jj) * d + rot(p, jj % 32, d)] =
                            h1[((size_t)hd * d + p) * h + r * q + jj];
    }
    if (cl_ok) {
        hw2.resize(src2.size());
        for (uint32_t hd = 0; hd < H; ++hd)
            for (uint32_t w = 0; w < W; ++w)
                for (uint32_t c = 0; c < 32; ++c)
                    for (uint32_t p = 0; p < rows2; ++p)
                        hw2[(((size_t)hd * W + w) * 32 + c) * rows2 + rot(p, c, rows2)] =
                            src2[((size_t)hd * rows2 + p) * L + c * W + w];
    }
    if (!up(&hs->w1, h1) || !up(&hs->b1, hb) || !up(&hs->w2, h2) || !up(&hs->w2_perm, hp) ||
        !up(&hs->w1_slices, hs1) || !up(&hs->w2_words, hw2)) {
        spl_hasher_destroy(hs);
        return fail(ctx, SPL_E_CUDA, "hasher: device allocation failed");
    }
    // tcgen05 bulk encoder operands (encode_tc.cu / spl_tc.cuh): per head, B
    // operands K-major bf16 swizzled: W1^T [N1 = h (linear: L)][K = d] and
    // W2^T [L][K = h]
    if (encode_tc_eligible(kind, d, h, L)) {
        const uint32_t N1 = kind == SPL_HASHER_MLP ? h : L, cols1 = N1;
        const size_t ob1 = tc_operand_bytes(N1), ob2 = tc_operand_bytes(L);
        std::vector<uint8_t> t1((size_t)H * ob1), t2(kind == SPL_HASHER_MLP ? (size_t)H * ob2 : 0);
        for (uint32_t hd = 0; hd < H; ++hd)
            for (uint32_t n = 0; n < N1; ++n)
                for (uint32_t k = 0; k < d; ++k) {
                    const uint16_t b = tc_bf16_bits(h1[((size_t)hd * d + k) * cols1 + n]);
                    std::memcpy(&t1[hd * ob1 + tc_sw_off(n, k, N1)], &b, 2);
                }
        if (kind == SPL_HASHER_MLP)
            for (uint32_t hd = 0; hd < H; ++hd)
                for (uint32_t n = 0; n < L; ++n)
                    for (uint32_t k = 0; k < h; ++k) {
                        const uint16_t b = tc_bf16_bits(h2[((size_t)hd * h + k) * L + n]);
                        std::memcpy(&t2[hd * ob2 + tc_sw_off(n, k, L)], &b, 2);
                    }
        auto upb = [&](void** dst, const std::vector<uint8_t>& src) -> bool {
            if (src.empty()) return true;
            if (cudaMalloc(dst, src.size()) != cudaSuccess) return false;
            return cudaMemcpy(*dst, src.data(), src.size(), cudaMemcpyHostToDevice) == cudaSuccess;
        };
        if (!upb(&hs->w1_tc, t1) || !upb(&hs->w2_tc, t2)) {
            spl_hasher_destroy(hs);
            return fail(ctx, SPL_E_CUDA, "hasher: device allocation failed");
        }
    }
    *out = hs;
    return SPL_OK;
}

void spl_hasher_destroy(spl_hasher* hs) {
    if (!hs) return;
    cudaFree(hs->w1);
    cudaFree(hs->b1);
    cudaFree(hs->w2);
    cudaFree(hs->w2_perm);
    cudaFree(hs->w1_slices);
    cudaFree(hs->w2_words);
    cudaFree(hs->w1_tc);
    cudaFree(hs->w2_tc);
    delete hs;
}

spl_status spl_mlp_forward(spl_ctx* ctx, const spl_hasher* hs, const float* x, uint32_t B,
                           uint32_t m, float* pre, void* stream) {
    if (!ctx || !hs) return SPL_E_STATE;
    EncJob j{};
    j.x = x;
    j.m = m;
    j.out_mode = ENC_PRE;
    j.pre = pre;
    return encode_exact_launch(ctx, hs, B, &j, 1, S(stream));
}

spl_status spl_encode(spl_ctx* ctx, const spl_hasher* hs, const float* x, uint32_t B, uint32_t m,
                      int mode, uint32_t* codes, void* stream) {
    NvtxRange nvtx_("spl_encode");
    if (!ctx || !hs) return SPL_E_STATE;
    if (mode == SPL_ENCODE_TC)
        return encode_tc_launch(ctx, hs, x, SPL_F32, B, m, codes, nullptr, S(stream));
    if (mode != SPL_ENCODE_EXACT) return fail(ctx, SPL_E_DIMENSION, "encode: unknown mode");
    EncJob j{};
    j.x = x;
    j.m = m;
    j.out_mode = ENC_CODES;
    j.codes = codes;
    return encode_exact_launch(ctx, hs, B, &j, 1, S(stream));
}

spl_status spl_encode_tc(spl_ctx* ctx, const spl_hasher* hs, const void* x, int x_dtype,
                         uint32_t B, uint32_t m, uint32_t* codes, float* pre, void* stream) {
    NvtxRange nvtx_("spl_encode_tc");
    if (!ctx || !hs) return SPL_E_STATE;
    return encode_tc_launch(ctx, hs, x, x_dtype, B, m, codes, pre, S(stream));
}

spl_status spl_encode_append(spl_ctx* ctx, const spl_hasher* hs, const float* k_new,
                             const float* v_new, uint32_t B, uint32_t* codes, void* kcache,
                             void* vcache, int kv_dtype, uint64_t cap, const uint32_t* pos,
                             void* stream) {
    NvtxRange nvtx_("spl_encode_append");
    if (!ctx || !hs) return SPL_E_STATE;
    if (kv_dtype != SPL_F32 && kv_dtype != SPL_BF16)
        return fail(ctx, SPL_E_DIMENSION, "encode_append: unknown kv dtype");
    EncJob j{};
    j.x = k_new;
    j.m = 1;
    j.out_mode = ENC_APPEND;
    j.codes = codes;
    j.cap = cap;
    j.pos = pos;
    j.v_new = v_new;
    j.kcache = kcache;
    j.vcache = vcache;
    j.kv_dtype = kv_dtype;
    return encode_exact_launch(ctx, hs, B, &j, 1, S(stream));
}

// ------------------------------------------------------------ attention
spl_status spl_sparse_attend(spl_ctx* ctx, const float* q, const void* kcache,
                             const void* vcache, int kv_dtype, uint64_t problem_stride_rows,
                             uint32_t d, uint32_t P, const uint32_t* idx, uint64_t idx_stride,
                             const uint32_t* cnt, const uint32_t* n_valid, uint32_t nvalid_div,
                             float scale, float* out, void* stream) {
    NvtxRange nvtx_("spl_sparse_attend");
    if (!ctx) return SPL_E_STATE;
    if (!(scale > 0.0f)) return fail(ctx, SPL_E_DIMENSION, "attention: scale must be positive");
    if (nvalid_div == 0) return fail(ctx, SPL_E_DIMENSION, "sparse_attend: nvalid_div == 0");
    AttParams prm{};
    prm.q = q;
    prm.kc = kcache;
    prm.vc = vcache;
    prm.stride_rows = problem_stride_rows;
    prm.d = d;
    prm.P = P;
    prm.idx = idx;
    prm.idx_stride = idx_stride;
    prm.cnt = cnt;
    prm.n_valid = n_valid;
    prm.nvalid_div = nvalid_div;
    prm.qscale = scale * kLog2e;
    prm.out = out;
    prm.partial_mode = 0;
    return sparse_attend_launch(ctx, prm, (uint32_t)idx_stride, kv_dtype, S(stream));
}

spl_status spl_sparse_attend_partial(spl_ctx* ctx, const float* q, const void* kcache,
                                     const void* vcache, int kv_dtype,
                                     uint64_t problem_stride_rows, uint32_t d, uint32_t P,
                                     const uint32_t* idx, uint64_t idx_stride,
                                     const uint32_t* cnt, const uint32_t* own_row,
                                     uint32_t nvalid_div, float scale, float* partials,
                                     void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (!(scale > 0.0f)) return fail(ctx, SPL_E_DIMENSION, "attention: scale must be positive");
    AttParams prm{};
    prm.q = q;
    prm.kc = kcache;
    prm.vc = vcache;
    prm.stride_rows = problem_stride_rows;
    prm.d = d;
    prm.P = P;
    prm.idx = idx;
    prm.idx_stride = idx_stride;
    prm.cnt = cnt;
    prm.own_row = own_row;
    prm.nvalid_div = nvalid_div ? nvalid_div : 1;
    prm.qscale = scale * kLog2e;
    prm.out = partials;
    prm.partial_mode = 1;
    return sparse_attend_launch(ctx, prm, (uint32_t)idx_stride, kv_dtype, S(stream));
}

spl_status spl_attend_combine(spl_ctx* ctx, const float* partials, uint32_t R, uint32_t P,
                              uint32_t d, float* out, void* stream) {
    if (!ctx) return SPL_E_STATE;
    return attend_combine_launch(ctx, partials, R, P, d, out, S(stream));
}

// ------------------------------------------------------------ decode step
// The attention kernels read K / V row slices with 8- and 16-byte loads
static bool kv_aligned(const void* k, const void* v) {
    return ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15u) == 0;
}

spl_status spl_decode_step(spl_ctx* ctx, const spl_hasher* hs, const float* q,
                           const float* k_new, const float* v_new, uint32_t B,
                           uint32_t* codes, void* kcache, void* vcache, int kv_dtype,
                           uint64_t cap, const uint32_t* n_valid, uint64_t n_max, uint32_t k,
                           float scale, uint32_t* idx, uint32_t* cnt, float* out, void* stream) {
    NvtxRange nvtx_("spl_decode_step");
    if (!ctx || !hs) return SPL_E_STATE;
    if (n_max > cap)
        return fail(ctx, SPL_E_DIMENSION,
                    "decode_step: n_max=" + std::to_string(n_max) + " exceeds the cache capacity " +
                        std::to_string(cap));
    const uint32_t H = hs->H, W = hs->L / 32, P = B * H;
    // query codes live in the context scratch
    spl_status st = ensure_buffer(ctx, &ctx->scratch, &ctx->scratch_bytes,
                                  (size_t)P * W * 4 + 4 * (size_t)B, false, S(stream),
                                  "decode_step");
    if (st) return st;
    uint32_t* qcodes = static_cast<uint32_t*>(ctx->scratch);
    // the appended key goes to slot n_valid[b] - 1 (its own token)
    EncJob jobs[2]{};
    jobs[0].x = k_new;
    jobs[0].m = 1;
    jobs[0].out_mode = ENC_APPEND;
    jobs[0].codes = codes;
    jobs[0].cap = cap;
    jobs[0].pos = n_valid;
    jobs[0].pos_minus_one = 1;
    jobs[0].v_new = v_new;
    jobs[0].kcache = kcache;
    jobs[0].vcache = vcache;
    jobs[0].kv_dtype = kv_dtype;
    jobs[1].x = q;
    jobs[1].m = 1;
    jobs[1].out_mode = ENC_CODES;
    jobs[1].codes = qcodes;
    (void)W;
    if ((st = encode_exact_launch(ctx, hs, B, jobs, 2, S(stream)))) return st;
    // retrieval and attention in one launch when the fused geometry applies
    // (L = d = 128, scores on chip): each K3 CTA attends the rows it selects
    bool done = false;
    if (!(scale > 0.0f)) return fail(ctx, SPL_E_DIMENSION, "attention: scale must be positive");
    if (kv_aligned(kcache, vcache) &&
        (st = hamming_topk_attend_impl(ctx, codes, cap, hs->L, qcodes, P, n_valid, H, n_max, k, idx,
                                       cnt, q, kcache, vcache, kv_dtype, hs->d, scale * kLog2e, out,
                                       S(stream), &done)))
        return st;
    if (done) return SPL_OK;
    // the selected K/V rows are prefetched into L2 by the select when they
    // fit it comfortably (config 2: 43 MB; flushed-L2 step 61.5 -> 59.4 us);
    // larger gathers would thrash L2, tiny ones (config 1) only pay latency
    const uint32_t row_bytes = hs->d * (kv_dtype == SPL_BF16 ? 2u : 4u);
    const uint64_t pf_bytes = (uint64_t)P * (k + 1) * row_bytes * 2;
    if (pf_bytes >= (4ull << 20) && pf_bytes <= (64ull << 20)) {
        ctx->k3_pf_k = kcache;
        ctx->k3_pf_v = vcache;
        ctx->k3_pf_row_bytes = row_bytes;
    }
    st = hamming_topk_impl(ctx, codes, cap, hs->L, qcodes, P, n_valid, H, n_max, k, idx, cnt,
                           S(stream));
    ctx->k3_pf_k = ctx->k3_pf_v = nullptr;
    ctx->k3_pf_row_bytes = 0;
    if (st) return st;
    return spl_sparse_attend(ctx, q, kcache, vcache, kv_dtype, cap, hs->d, P, idx, k, cnt,
                             n_valid, H, scale, out, stream);
}

spl_status spl_sharded_decode_step(spl_ctx* ctx, spl_peer* peer, const spl_hasher* hs,
                                   const float* q, const float* k_new, const float* v_new,
                                   uint32_t B, int owner, uint32_t* codes, void* kcache,
                                   void* vcache, int kv_dtype, uint64_t cap,
                                   const uint32_t* n_valid, uint64_t n_max, uint32_t k, float scale,
                                   uint32_t* idx, uint32_t* cnt, uint32_t* out_offset, float* out,
                                   void* stream) {
    NvtxRange nvtx_("spl_sharded_decode_step");
    if (!ctx || !hs || !peer) return SPL_E_STATE;
    if (!peer->connected) return fail(ctx, SPL_E_STATE, "sharded_decode_step: peer group not connected");
    if (!(scale > 0.0f)) return fail(ctx, SPL_E_DIMENSION, "attention: scale must be positive");
    if (!kv_aligned(kcache, vcache))
        return fail(ctx, SPL_E_DIMENSION, "sharded_decode_step: K / V caches must be 16-byte aligned");
    if (n_max > cap)
        return fail(ctx, SPL_E_DIMENSION,
                    "sharded_decode_step: n_max=" + std::to_string(n_max) +
                        " exceeds the cache capacity " + std::to_string(cap));
    const uint32_t H = hs->H, W = hs->L / 32, P = B * H;
    spl_status st = ensure_buffer(ctx, &ctx->scratch, &ctx->scratch_bytes,
                                  (size_t)P * W * 4 + 4 * (size_t)B, false, S(stream),
                                  "sharded_decode_step");
    if (st) return st;
    uint32_t* qcodes = static_cast<uint32_t*>(ctx->scratch);
    // every workspace of the step is sized before its first launch: the
    // retrieval kernel waits for the peers inside, and an allocation (or a
    // zero-fill synchronisation) behind it would stall the group
    if ((st = reserve_impl(ctx, P, n_max, hs->L, k, hs->d, S(stream)))) return st;
    // every rank encodes the query; the rank the new token belongs to appends it
    EncJob jobs[2]{};
    int nj = 0;
    if (owner) {
        jobs[nj].x = k_new;
        jobs[nj].m = 1;
        jobs[nj].out_mode = ENC_APPEND;
        jobs[nj].codes = codes;
        jobs[nj].cap = cap;
        jobs[nj].pos = n_valid;
        jobs[nj].pos_minus_one = 1;
        jobs[nj].v_new = v_new;
        jobs[nj].kcache = kcache;
        jobs[nj].vcache = vcache;
        jobs[nj].kv_dtype = kv_dtype;
        ++nj;
    }
    jobs[nj].x = q;
    jobs[nj].m = 1;
    jobs[nj].out_mode = ENC_CODES;
    jobs[nj].codes = qcodes;
    ++nj;
    if ((st = encode_exact_launch(ctx, hs, B, jobs, nj, S(stream)))) return st;
    bool done = false;
    if ((st = hamming_topk_attend_impl(ctx, codes, cap, hs->L, qcodes, P, n_valid, H, n_max, k, idx,
                                       cnt, q, kcache, vcache, kv_dtype, hs->d, scale * kLog2e, out,
                                       S(stream), &done, peer, out_offset, owner)))
        return st;
    if (done) return SPL_OK;
    // unfused: sharded retrieval, this rank's partial attention, peer combine
    if ((st = hamming_topk_sharded_impl(ctx, peer, codes, cap, hs->L, qcodes, P, n_valid, H, n_max,
                                        k, idx, cnt, out_offset, S(stream))))
        return st;
    const uint32_t d = hs->d;
    st = ensure_buffer(ctx, &ctx->dense_ws, &ctx->dense_ws_bytes, (size_t)P * (d + 2) * sizeof(float),
                       false, S(stream), "sharded_decode_step");
    if (st) return st;
    float* part = static_cast<float*>(ctx->dense_ws);
    AttParams prm{};
    prm.q = q;
    prm.kc = kcache;
    prm.vc = vcache;
    prm.stride_rows = cap;
    prm.d = d;
    prm.P = P;
    prm.idx = idx;
    prm.idx_stride = k;
    prm.cnt = cnt;
    prm.n_valid = n_valid;
    prm.nvalid_div = H;
    prm.own_row = nullptr;  // not the owner: no own row
    prm.own_nvalid = owner ? 1 : 0;
    prm.qscale = scale * kLog2e;
    prm.out = part;
    prm.partial_mode = 1;
    if ((st = sparse_attend_launch(ctx, prm, k, kv_dtype, S(stream)))) return st;
    return peer_combine_launch(ctx, peer, part, P, d, out, S(stream));
}

spl_status spl_budget_from_rate(double rate, uint64_t n, uint32_t* k) {
    if (!k) return SPL_E_STATE;
    if (!(rate > 0.0 && rate <= 1.0)) return SPL_E_DIMENSION;
    const uint32_t raw = (uint32_t)(rate * (double)n);
    const uint64_t kk = raw > 20 ? raw : 20;
    *k = (uint32_t)(kk < n ? kk : n);
    return SPL_OK;
}

}  // extern "C"
