// Internal shared definitions for the sm_100a kernels behind include/spl_c.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/spl_c.h"

#define SPL_DEV_ERR_NUMERIC 1u
#define SPL_DEV_ERR_DIMENSION 2u
#define SPL_DEV_ERR_STALL 4u  // K3-fused watchdog: a problem's CTAs were not co-resident

// One context per caller (see spl_c.h). Owns the workspace and the device
// error word. Workspace regions are sized by spl_reserve or lazily (never
// during stream capture).
struct spl_ctx {
    int device = 0;
    int num_sms = 148;        // SMs this context can use (see usable_sms in capi.cu)
    bool k3_coop = false;     // SM-limited context: fused K3 launches are cooperative
    std::string err;
    uint64_t launches = 0;
    std::string launch_log;  // kernel names since the last spl_launch_log (bounded)
    double last_train_loop_ms = 0.0;  // device time of the last spl_train_hasher loop
    // decode step: K/V caches whose selected rows the K3 select prefetches
    // into L2 for K4 (set by spl_decode_step when the gathered rows fit L2)
    const void* k3_pf_k = nullptr;
    const void* k3_pf_v = nullptr;
    uint32_t k3_pf_row_bytes = 0;

    uint32_t* dev_err = nullptr;  // device error word (bit flags above)

    // K3 workspace: scores + segment records + per-segment plans.
    void* k3_ws = nullptr;
    size_t k3_ws_bytes = 0;
    // K3 per-problem persistent state, zero between launches (self-resetting):
    // counters[P] + total histograms [P][Lmax+2].
    uint32_t* k3_state = nullptr;
    size_t k3_state_words = 0;

    // K4 workspace: partials [P][splits][d+2] + per-problem counters.
    float* att_ws = nullptr;
    size_t att_ws_bytes = 0;
    uint32_t* att_counters = nullptr;
    size_t att_counters_n = 0;

    // dense retrieval (oracle_topk) logits [P][n_max] when the caller passes none.
    void* dense_ws = nullptr;
    size_t dense_ws_bytes = 0;

    // generic scratch for encoders / top_k keys.
    void* scratch = nullptr;
    size_t scratch_bytes = 0;

    // last shard-histogram geometry (the select phase reuses its records).
    uint64_t shard_n_max = 0;
    uint32_t shard_P = 0, shard_L = 0, shard_G = 0;
    uint64_t shard_S = 0;
};

// A sequence-sharding peer group member (fused in-kernel exchange, see
// hamming_topk.cu "peer exchange"): this rank's exchange area, the table of
// every rank's area as mapped into this process, and the call epoch.
struct spl_peer {
    uint32_t R = 0, rank = 0, Pmax = 0, Lmax = 0;
    uint32_t* buf = nullptr;        // own exchange area (zeroed at creation)
    size_t bytes = 0;
    uint32_t** d_table = nullptr;   // [R] device pointers (own included)
    std::vector<void*> opened;      // IPC mappings to close
    uint32_t* d_epoch = nullptr;    // call counter (device, so graph replays advance it)
    bool connected = false;
    int device = 0;
};

struct spl_hasher {
    int kind = SPL_HASHER_MLP;
    uint32_t H = 0, d = 0, h = 0, L = 0;
    float* w1 = nullptr;  // [H][d][h]  (linear: projection [H][d][L])
    float* b1 = nullptr;  // [H][h]
    float* w2 = nullptr;  // [H][h][L]
    float* w2_perm = nullptr;  // layer 2 (linear: projection) columns permuted, see capi.cu
    float* w1_slices = nullptr;  // [H][4][h/4][d] column quarters of W1, row per output (cluster encoder)
    float* w2_words = nullptr;   // [H][W][32][act_dim] word-major layer 2, row per output (cluster encoder)
    // bf16 copies for the tcgen05 bulk encoder (K-major packing, see encode_tc.cu)
    void* w1_tc = nullptr;
    void* w2_tc = nullptr;
};

namespace spl {

inline spl_status fail(spl_ctx* ctx, spl_status st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return st;
}

inline spl_status cuda_fail(spl_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, SPL_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define SPL_CUDA_TRY(ctx, expr)                                          \
    do {                                                                 \
        cudaError_t _e = (expr);                                         \
        if (_e != cudaSuccess) return ::spl::cuda_fail((ctx), _e, #expr); \
    } while (0)

// After a launch: count it, surface launch-config errors.
inline spl_status after_launch(spl_ctx* ctx, const char* name) {
    ctx->launches++;
    if (ctx->launch_log.size() < 4096) {
        ctx->launch_log += name;
        ctx->launch_log += ';';
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, name);
    return SPL_OK;
}

// Programmatic dependent launch (PDL) along the decode chain K1 -> K3 -> K4
// -> K1 ...: each kernel lets its dependent launch as soon as all of its own
// CTAs are running (pdl_trigger at entry — the dependent is released only
// when every CTA of this grid has triggered, so co-residency assumptions of
// this grid are never undercut), and waits for its predecessor's completion
// and memory (pdl_wait) right before it first reads or writes shared data.
// Prologues (weight TMA, counter zeroing) overlap the predecessor's tail.
// Without the launch attribute both are no-ops. Opt-in (SPL_PDL=1): see
// pdl_enabled() for the measurement that keeps it off by default.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       void** args);

inline bool stream_capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) return false;
    return st != cudaStreamCaptureStatusNone;
}

// Grow a device buffer to at least `bytes` (zero-filled when `zero`).
spl_status ensure_buffer(spl_ctx* ctx, void** buf, size_t* have, size_t bytes, bool zero,
                         cudaStream_t s, const char* what);

__device__ __forceinline__ void raise_dev_err(uint32_t* e, uint32_t flag) {
    if (e) atomicOr(e, flag);
}

}  // namespace spl
