#!/usr/bin/env python
"""Benchmark of the Spotlight decode-time retrieval path on B200.

Headline (BASELINE.json `metric`, config 3): Hamming top-k retrieval over a
512K-token x 32-head cache of 128-bit codes, k = budget_from_rate(0.02) =
10485, one retrieval = K3 scan + select (spl_hamming_topk), inputs resident in
HBM (268 MB of codes per step > 126 MB L2, so no L2 flush is needed). `value`
is the device time per retrieval in microseconds (max over ranks; lower is
better).  For N > 1 GPUs the cache is sequence-sharded (config 5, weak
scaling: 512K tokens per GPU, total N x 512K): local scan + histogram, NCCL
all-gather of the [32][129] histograms, global threshold + tie quota, local
ordered select.

Secondary (config 2): one full decode step of a 32-head layer at 128K context
(encode-append of the new key + query encode + retrieval + sparse attention
over bf16 K/V) -> sparse decode tok/s.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libspotref.so = the unmodified reference sources, else the C
port) on the same workload on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "Hamming top-k retrieval µs @512K tokens (HBM GB/s %peak); sparse decode tok/s"
H, N_TOK, L, D = 32, 524288, 128, 128


def peaks():
    try:
        p = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def tensor_peak():
    """(burst, sustained) dense bf16 TF/s from MEASURED_PEAKS.json."""
    try:
        p = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(p["bf16_tflops"]), float(p["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 2250.0, 2250.0, "fallback (nominal dense)"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- inputs
def random_codes(torch, P, n, W, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    return torch.randint(-2**31, 2**31 - 1, (P, n, W), generator=g, device=dev, dtype=torch.int32)


def event_timer(torch, fn, steps, stream):
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for _ in range(steps):
        fn()
    end.record(stream)
    torch.cuda.synchronize()
    return start.elapsed_time(end) / steps  # ms per step


_FLUSH = {}


def flushed_timer(torch, fn, steps, stream):
    """Median per-call ms with L2 flushed before every call, outside the timed
    window: a 512 MB write (> the 126 MB L2) followed by a 256 MB read, so the
    dirty lines of the write are written back before the call and L2 holds
    only clean, unrelated lines. For working sets that would otherwise stay
    L2-resident across back-to-back steps."""
    if "buf" not in _FLUSH:
        _FLUSH["buf"] = torch.empty((512 << 20) // 4, dtype=torch.int32, device="cuda")
        _FLUSH["rd"] = torch.ones((256 << 20) // 4, dtype=torch.int32, device="cuda")
        _FLUSH["acc"] = torch.zeros(1, dtype=torch.int64, device="cuda")
    buf, rd, acc = _FLUSH["buf"], _FLUSH["rd"], _FLUSH["acc"]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    torch.cuda.synchronize()
    for a, b in evs:
        buf.fill_(1)
        acc.add_(rd.sum())
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def flushed_graph_timer(torch, fn, steps, warmup):
    """Device ms per call with L2 flushed before every call and without the
    per-launch host/driver gap: one CUDA graph holds `steps` x (flush, call),
    a second one the same `steps` flushes alone; both are timed with CUDA
    events around a replay, and the difference / steps is the call's device
    time (the flush = a 512 MB write then a 256 MB read, so L2 holds only
    clean unrelated lines when the call starts). Returns (ms, flush_ms) or
    None if capture fails."""
    if "buf" not in _FLUSH:
        flushed_timer(torch, lambda: None, 1, torch.cuda.current_stream())
    buf, rd, acc = _FLUSH["buf"], _FLUSH["rd"], _FLUSH["acc"]

    def flush():
        buf.fill_(1)
        acc.add_(rd.sum())
    try:
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        g1, g0 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=gs, capture_error_mode="relaxed"):
            for _ in range(steps):
                flush()
                fn(gs)
        with torch.cuda.graph(g0, stream=gs, capture_error_mode="relaxed"):
            for _ in range(steps):
                flush()
        cur = torch.cuda.current_stream()
        for _ in range(max(1, warmup // 2)):
            g1.replay()
            g0.replay()
        torch.cuda.synchronize()
        t1 = min(event_timer(torch, g1.replay, 1, cur) for _ in range(3))
        t0 = min(event_timer(torch, g0.replay, 1, cur) for _ in range(3))
        del g1, g0
        return (t1 - t0) / steps, t0 / steps
    except Exception:
        return None


def graph_timer(torch, fn, steps, warmup, flush=False):
    """Capture one call of fn (our kernels on a side stream) in a CUDA graph
    and time `steps` replays; None if capture is not possible. flush: L2
    flushed before every replay (flushed_timer)."""
    try:
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs, capture_error_mode="relaxed"):
            fn(gs)
        for _ in range(warmup):
            graph.replay()
        torch.cuda.synchronize()
        if flush:
            return flushed_timer(torch, graph.replay, steps, torch.cuda.current_stream())
        return event_timer(torch, graph.replay, steps, torch.cuda.current_stream())
    except Exception:
        return None


# ---------------------------------------------------------------- CPU legs
def cpu_reference_retrieval(codes_np, q_np, k, threads, reps, warmup):
    """The reference's retrieval (per head nxor_scores_into + top_k_indices,
    heads over OpenMP threads) on host cores. Returns (us per retrieval list,
    kind, result of the last run)."""
    from oracle_lib import Oracle, RefLib

    P, n, W = codes_np.shape
    nv = np.full(P, n, np.uint32)
    times = []
    out = None
    if RefLib.available():
        ref = RefLib()
        h = ref.index_create(codes_np, nv)
        try:
            for i in range(warmup + reps):
                t0 = time.perf_counter()
                out = ref.retrieve_batch(h, q_np, nv, k, threads)
                dt = (time.perf_counter() - t0) * 1e6
                if i >= warmup:
                    times.append(dt)
        finally:
            ref.index_destroy(h)
        return times, "reference", out
    orc = Oracle()
    for i in range(warmup + reps):
        t0 = time.perf_counter()
        out = orc.retrieve_batch(codes_np, q_np, nv, k, threads)
        dt = (time.perf_counter() - t0) * 1e6
        if i >= warmup:
            times.append(dt)
    return times, "port", out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # the same workload as our arm: N x 512K tokens per head at N GPUs
    # (config 5 when N > 1), k = 2% of the whole cache
    world = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    n_tot = N_TOK * world
    rng = np.random.default_rng(0)
    codes = rng.integers(0, 2**32, (H, n_tot, L // 32), dtype=np.uint32)
    q = rng.integers(0, 2**32, (H, L // 32), dtype=np.uint32)
    k = budget(n_tot)
    steps = args.steps if world == 1 else min(args.steps, 10)  # bounded sample
    times, kind, _ = cpu_reference_retrieval(codes, q, k, threads, steps, args.warmup)
    v = statistics.mean(times)
    line = {"metric": METRIC, "value": round(v, 2), "unit": "µs", "impl": "reference",
            "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": round(v / 1000, 4), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": workload_config(world),
            "cpu_baseline": {"value": round(v, 2), "unit": "µs", "cores": threads, "kind": kind,
                             "sample": f"full workload per step ({H} heads x {n_tot} rows: per head "
                                       f"nxor_scores_into + top_k_indices), heads spread over "
                                       f"{threads} OpenMP threads"},
            "e2e": {"value": round(v, 2), "unit": "µs", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def budget(n):
    return min(max(int(0.02 * n), 20), n)


def workload_config(world):
    """The `config` of the JSON line — identical in both arms (ours and
    --impl reference) so the driver can match them."""
    n_total = N_TOK * world
    k = budget(n_total)
    return {"workload": ("config3: 32 heads x 524288 tokens x 128-bit codes, k=10485" if world == 1 else
                         f"config5: sequence-sharded {n_total} tokens x 32 heads x 128-bit codes, "
                         f"k={k}, per-head histograms exchanged across ranks"),
            "heads": H, "tokens_per_gpu": N_TOK, "tokens_total": n_total, "code_bits": L, "k": k,
            "l2": "inputs (268 MB of codes per GPU) larger than the 126 MB L2; value without flush, "
                  "value_l2_flushed with L2 flushed before every retrieval"}


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    from paper_2508_19740_b200 import capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SPL_BENCH_SAME_GPU=1: every rank on GPU 0 with gloo collectives (host
    # staged) — exercises the N > 1 code paths on a one-GPU box (timings are
    # then meaningless: the ranks time-share the GPU)
    same_gpu = os.environ.get("SPL_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        dist = dist_mod
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def all_gather_dev(out, inp):
        if not same_gpu:
            dist.all_gather_into_tensor(out, inp)
            return
        parts = [torch.empty_like(inp, device="cpu") for _ in range(world)]
        dist.all_gather(parts, inp.cpu())
        out.copy_(torch.stack(parts).to(dev))

    def all_reduce_dev(t, op):
        if not same_gpu:
            dist.all_reduce(t, op=op)
            return
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c.to(dev))
    ctx = capi.Context(local)
    stream = torch.cuda.current_stream()
    W = L // 32
    P = H
    n_local = N_TOK  # weak scaling: 512K tokens per GPU
    n_total = n_local * world
    k = budget(n_total)

    codes = random_codes(torch, P, n_local, W, seed=1234 + rank, dev=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(99)
    qcodes = torch.randint(-2**31, 2**31 - 1, (P, W), generator=g, device=dev, dtype=torch.int32)
    nvalid = torch.full((P,), n_local, dtype=torch.int32, device=dev)
    idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros(P, dtype=torch.int32, device=dev)
    off = torch.zeros(P, dtype=torch.int32, device=dev)
    hist = torch.zeros((P, L + 1), dtype=torch.int32, device=dev)
    all_hist = torch.zeros((world, P, L + 1), dtype=torch.int32, device=dev)

    shard_path = None
    if world == 1:
        def retrieval():
            ctx.hamming_topk(codes, n_local, L, qcodes, P, nvalid, 1, n_local, k, idx, cnt, stream)
    else:
        def retrieval_nccl():
            ctx.shard_histogram(codes, n_local, L, qcodes, P, nvalid, 1, n_local, hist, stream)
            all_gather_dev(all_hist, hist)
            ctx.shard_select(all_hist, world, rank, L, P, nvalid, 1, n_local, k, idx, cnt, off, stream)

        # Fused path: one kernel per rank, the histogram exchange inside it over
        # NVLink peer memory (IPC-mapped exchange areas). Checked once against
        # the two-kernel NCCL flow on every rank; any mismatch or error keeps
        # the NCCL flow for the timed run.
        retrieval = retrieval_nccl
        shard_path = "nccl (k3_scan + all-gather + k3_shard_plan + k3_select)"

        def agree(flag):  # every rank takes the same branch
            t = torch.tensor([1 if flag else 0], device=dev)
            all_reduce_dev(t, dist.ReduceOp.MIN)
            return int(t.item()) == 1

        peer, err = None, None
        try:
            peer = ctx.peer(world, rank, P, L)
            handles = [None] * world
            dist.all_gather_object(handles, peer.ipc_handle())
            if os.environ.get("SPL_BENCH_FAIL_PEER_RANK") == str(rank):  # test hook: one-sided failure
                raise RuntimeError("injected peer-open failure")
            peer.open(handles)
        except Exception as e:  # no IPC / peer access: keep the NCCL flow
            err = str(e)[:60]
        if agree(err is None):
            def retrieval_fused():
                ctx.hamming_topk_sharded(peer, codes, n_local, L, qcodes, P, nvalid, 1, n_local, k,
                                         idx, cnt, off, stream)
            retrieval_nccl()
            torch.cuda.synchronize()
            ref = (idx.clone(), cnt.clone(), off.clone())
            dist.barrier()
            same = False
            try:
                retrieval_fused()
                torch.cuda.synchronize()
                ctx.check_device_error()
                same = all(torch.equal(a, b) for a, b in zip(ref, (idx, cnt, off)))
            except Exception as e:
                err = str(e)[:60]
            if agree(same):
                retrieval = retrieval_fused
                shard_path = "fused (one k3_fused<SHARD> per rank, in-kernel exchange over NVLink peer memory)"
            else:
                shard_path = f"nccl (fused path {'failed: ' + err if err else 'disagreed with it on this run'})"
        else:
            shard_path = f"nccl (fused path unavailable: {err or 'on another rank'})"

    for _ in range(args.warmup):
        retrieval()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    l0 = ctx.launches()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    eager_ms = event_timer(torch, retrieval, args.steps, stream)
    launches = ctx.launches() - l0
    ms = eager_ms
    # Decode loops replay a captured CUDA graph: capture one retrieval and time
    # exactly `steps` replays (the same device work, without per-call host
    # launch latency between back-to-back steps).
    graph_note = None
    per_replay_ms = None
    if world == 1:
        try:
            gs = torch.cuda.Stream()
            gs.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=gs, capture_error_mode="relaxed"):
                ctx.hamming_topk(codes, n_local, L, qcodes, P, nvalid, 1, n_local, k, idx, cnt, gs)
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()
            per_replay_ms = event_timer(torch, graph.replay, args.steps, torch.cuda.current_stream())
            del graph
            # A decode loop captures its whole step sequence in one graph:
            # `steps` retrievals back to back in ONE graph, replayed once and
            # timed as a whole (K dependent launches on one stream, each a
            # full retrieval; the per-replay host/driver gap of the form
            # above, ~3 us, is not part of the retrieval).
            gk = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gk, stream=gs, capture_error_mode="relaxed"):
                for _ in range(args.steps):
                    ctx.hamming_topk(codes, n_local, L, qcodes, P, nvalid, 1, n_local, k, idx, cnt, gs)
            gk.replay()
            torch.cuda.synchronize()
            ms = statistics.median(event_timer(torch, gk.replay, 1, torch.cuda.current_stream())
                                   for _ in range(3)) / args.steps
            del gk
            graph_note = (f"one CUDA graph of {args.steps} back-to-back retrievals, replayed once "
                          f"(median of 3 replays) / {args.steps}")
        except Exception as e:  # capture unsupported: keep the eager number
            graph_note = f"eager (graph capture failed: {str(e)[:80]})"
    elif shard_path and shard_path.startswith("fused"):
        # the fused sharded retrieval has no host collective inside: every
        # rank captures `steps` of them in one graph and replays it at the
        # same time (the kernels meet through peer memory), as at N = 1
        gk, err = None, None
        try:
            gs = torch.cuda.Stream()
            gs.wait_stream(torch.cuda.current_stream())
            gk = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gk, stream=gs, capture_error_mode="relaxed"):
                for _ in range(args.steps):
                    ctx.hamming_topk_sharded(peer, codes, n_local, L, qcodes, P, nvalid, 1, n_local, k,
                                             idx, cnt, off, gs)
        except Exception as e:
            err = str(e)[:80]
        if agree(err is None):
            dist.barrier()
            gk.replay()
            torch.cuda.synchronize()
            res = []
            for _ in range(3):
                dist.barrier()
                res.append(event_timer(torch, gk.replay, 1, torch.cuda.current_stream()) / args.steps)
            ctx.check_device_error()
            ms = statistics.median(res)
            graph_note = (f"one CUDA graph of {args.steps} back-to-back sharded retrievals per rank, "
                          "replayed together (median of 3) / steps, max over ranks")
        else:
            graph_note = f"eager (graph capture failed: {err or 'on another rank'})"
        del gk
    # the same retrieval with L2 flushed before every call (device time from
    # CUDA graphs of steps x (flush, call) minus steps x flush): the inputs
    # already exceed L2, this shows the number does not lean on L2 residue
    flushed_ms = None
    if world == 1:
        fl = flushed_graph_timer(
            torch, lambda st: ctx.hamming_topk(codes, n_local, L, qcodes, P, nvalid, 1, n_local, k, idx,
                                               cnt, st), min(args.steps, 20), args.warmup)
        flushed_ms = fl[0] if fl else None
    if dist:
        t = torch.tensor([ms], device=dev)
        all_reduce_dev(t, dist.ReduceOp.MAX)
        ms = float(t.item())
    us = ms * 1000.0

    # scan-kernel share: the same streaming kernel alone (shard mode, no select)
    def scan_only():
        ctx.shard_histogram(codes, n_local, L, qcodes, P, nvalid, 1, n_local, hist, stream)
    for _ in range(3):
        scan_only()
    scan_ms = event_timer(torch, scan_only, args.steps, stream)

    # e2e through the C-ABI with host buffers: H2D of the step's query vectors
    # (encoded on device, exact mode), retrieval, D2H of the indices + counts.
    # (N > 1: every rank encodes the step's queries, runs the sharded flow and
    # reads back its share of the indices + their global offsets)
    rng = np.random.default_rng(7)
    decode = None
    decode4 = None
    prefill = None
    accuracy = None
    train = None
    config1 = None
    w1 = (rng.standard_normal((H, D, D)) / np.sqrt(D)).astype(np.float32)
    b1 = np.zeros((H, D), np.float32)
    w2 = (rng.standard_normal((H, D, L)) / np.sqrt(D)).astype(np.float32)
    hasher = ctx.hasher(w1, b1, w2)
    q_host = torch.from_numpy(rng.standard_normal((1, H, D)).astype(np.float32)).pin_memory()
    idx_host = torch.empty((P, k), dtype=torch.int32).pin_memory()
    cnt_host = torch.empty(P, dtype=torch.int32).pin_memory()
    off_host = torch.empty(P, dtype=torch.int32).pin_memory()
    q_dev = torch.empty((1, H, D), dtype=torch.float32, device=dev)

    def e2e_step():
        q_dev.copy_(q_host, non_blocking=True)
        hasher.encode(q_dev, 1, 1, qcodes, capi.SPL_ENCODE_EXACT, stream)
        retrieval()
        idx_host.copy_(idx, non_blocking=True)
        cnt_host.copy_(cnt, non_blocking=True)
        if world > 1:
            off_host.copy_(off, non_blocking=True)

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e2e_ms = event_timer(torch, e2e_step, args.steps, stream)
    e2e_serial_ms = e2e_ms
    e2e_note = "serial: every copy and kernel of a step on one stream"
    if world == 1:
        # The serving form of the same loop (independent queries, software-
        # pipelined across steps): step i is one CUDA graph that runs
        # retrieval(i) and, on two parallel branches, the D2H of step i-1's
        # indices and the H2D + exact encode of step i+1's query (query
        # vectors, codes and index buffers double-buffered), so the read-back
        # and the next encode overlap the retrieval (the encode runs on the
        # SMs the retrieval's last CTAs leave free). Every step still pays its
        # own H2D, encode, retrieval and D2H inside the timed region, which
        # starts with step 0's H2D + encode and ends with the last D2H.
        try:
            gs, cps, cs2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
            gs.wait_stream(stream)
            idx_b = [idx, torch.empty_like(idx)]
            cnt_b = [cnt, torch.empty_like(cnt)]
            idx_hb = [idx_host, torch.empty_like(idx_host).pin_memory()]
            cnt_hb = [cnt_host, torch.empty_like(cnt_host).pin_memory()]
            q_b = [q_dev, torch.empty_like(q_dev)]
            qc_b = [qcodes, torch.empty_like(qcodes)]

            def d2h(b):
                idx_hb[b].copy_(idx_b[b], non_blocking=True)
                cnt_hb[b].copy_(cnt_b[b], non_blocking=True)

            def encode_next(b, st):
                q_b[b].copy_(q_host, non_blocking=True)
                hasher.encode(q_b[b], 1, 1, qc_b[b], capi.SPL_ENCODE_EXACT, st)

            graphs = []
            for b in range(2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=gs, capture_error_mode="relaxed"):
                    fork = torch.cuda.Event()
                    fork.record(gs)
                    cps.wait_event(fork)
                    cs2.wait_event(fork)
                    with torch.cuda.stream(cps):
                        d2h(1 - b)  # the previous step's result
                    with torch.cuda.stream(cs2):
                        encode_next(1 - b, cs2)  # the next step's query
                    ctx.hamming_topk(codes, n_local, L, qc_b[b], P, nvalid, 1, n_local, k, idx_b[b], cnt_b[b],
                                     gs)
                    for st in (cps, cs2):
                        join = torch.cuda.Event()
                        join.record(st)
                        gs.wait_event(join)
                graphs.append(g)

            def e2e_pipe(nsteps):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                encode_next(0, stream)  # step 0's H2D + encode
                for i in range(nsteps):
                    graphs[i & 1].replay()
                d2h((nsteps - 1) & 1)  # the last step's result
                e1.record(stream)
                torch.cuda.synchronize()
                return e0.elapsed_time(e1) / nsteps

            e2e_pipe(max(3, args.warmup))
            e2e_ms = min(e2e_pipe(args.steps) for _ in range(3))
            last = (args.steps - 1) & 1
            assert torch.equal(idx_hb[last], idx_b[last].cpu()) and torch.equal(idx_b[last], idx_b[1 - last])
            e2e_note = ("software-pipelined over independent queries, one CUDA graph per step: retrieval(i) with "
                        "step i-1's D2H and step i+1's H2D + encode on parallel branches (double-buffered); "
                        "the region starts with step 0's H2D + encode and ends with the last step's D2H")
        except Exception as e:  # keep the serial figure
            e2e_note = f"serial (pipelined form unavailable: {str(e)[:80]})"
    enc_ms = event_timer(torch, lambda: hasher.encode(q_dev, 1, 1, qcodes, capi.SPL_ENCODE_EXACT, stream),
                         args.steps, stream)
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        all_reduce_dev(t, dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    d2h = idx_host.numel() * 4 + cnt_host.numel() * 4 + (off_host.numel() * 4 if world > 1 else 0)
    e2e = {"value": round(e2e_ms * 1000, 2), "unit": "µs",
           "h2d_bytes_per_step": int(q_host.numel() * 4),
           "d2h_bytes_per_step": int(d2h),
           "path": ("spl_encode(query, exact) + spl_hamming_topk, pinned host buffers" if world == 1
                    else "spl_encode(query, exact) + " + (shard_path or "") +
                         ", pinned host buffers (max over ranks)"),
           "encode_us": round(enc_ms * 1000, 2),
           "schedule": e2e_note, "serial_us": round(e2e_serial_ms * 1000, 2)}
    sharded = heads = None
    if not args.no_decode:
        sharded = bench_sharded_decode(torch, capi, ctx, dev, stream, args, world, rank, dist, same_gpu,
                                       all_reduce_dev)
        if world > 1:
            heads = bench_head_sharded(torch, capi, ctx, dev, stream, args, world, rank, dist, same_gpu,
                                       all_reduce_dev)
    if world == 1:
        if not args.no_decode:
            decode = bench_decode(torch, capi, ctx, dev, stream, args, hasher)
        if not args.no_prefill:
            prefill = bench_prefill(torch, capi, ctx, dev, stream, args)
        if not args.no_decode:
            decode4 = bench_decode4(torch, capi, ctx, dev, stream, args)
        if not args.no_decode:
            accuracy = bench_accuracy(torch, capi, ctx, dev, stream, args)
        if not args.no_train:
            train = bench_train(capi, ctx, args)
        if not args.no_decode:
            config1 = bench_config1(torch, capi, ctx, dev, stream, args)
    clk = clocks.stop()

    # CPU baseline (rank 0, N = 1): the reference on this host's cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        codes_np = codes.cpu().numpy().view(np.uint32)
        q_np = qcodes.cpu().numpy().view(np.uint32)
        threads = os.cpu_count() or 1
        times, kind, ref_out = cpu_reference_retrieval(codes_np, q_np, k, threads, reps=3, warmup=1)
        hamming_topk_np = idx.cpu().numpy().view(np.uint32)
        ctx.hamming_topk(codes, n_local, L, qcodes, P, nvalid, 1, n_local, k, idx, cnt, stream)
        torch.cuda.synchronize()
        parity = bool(np.array_equal(idx.cpu().numpy().view(np.uint32), ref_out))
        cpu = {"value": round(statistics.mean(times), 1), "unit": "µs", "cores": threads,
               "kind": kind, "sample": f"3 full config-3 retrievals ({H} heads x {n_local} rows, "
                                       f"k={k}) after 1 warm-up; heads over {threads} threads",
               "gpu_indices_equal_reference": parity}
        # "as shipped": the reference's own loop is single-threaded for scan +
        # top-k (it only threads matmul); one full retrieval on one core
        t1, _, _ = cpu_reference_retrieval(codes_np, q_np, k, 1, reps=1, warmup=0)
        cpu["as_shipped_one_core"] = {"value": round(t1[0], 1), "unit": "µs", "cores": 1}
        del hamming_topk_np

    hbm, peak_kind = peaks()
    alg_bytes = P * n_local * W * 4 + P * W * 4 + P * k * 4  # SURVEY 8(d), per rank
    achieved = alg_bytes / (us * 1e-6) / 1e9
    scan_bytes = P * n_local * W * 4
    # dram bytes per retrieval: ncu cannot run inside the timed process, so
    # this is the newest committed ncu capture of the same kernel on the same
    # workload (caches flushed by ncu), stamped with the commit it was taken at
    traffic = traffic_src = traffic_b2b = None
    for tpath in sorted((ROOT / "profiles").glob("r*_k3_traffic.json"), reverse=True):
        try:
            tj = json.loads(tpath.read_text())
            traffic = tj.get("bytes_per_retrieval")
            traffic_src = f"{tpath.relative_to(ROOT)} (commit {tj.get('commit', 'unrecorded')})"
            # back-to-back retrievals (the `value` timing) read part of the
            # codes from L2: DRAM bytes per retrieval in that state
            traffic_b2b = (tj.get("back_to_back") or {}).get("dram_bytes_read_median")
            break
        except Exception:
            continue
    line = {
        "metric": METRIC, "value": round(us, 2), "unit": "µs", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": workload_config(world),
        "roofline": {"bound": "hbm",
                     "kernel": ("one retrieval = k3_fused (single launch)" if world == 1
                                else shard_path),
                     "achieved": round(achieved, 1), "peak": hbm, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "algorithmic_bytes": alg_bytes, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "traffic_back_to_back_dram_read": traffic_b2b,
                     "scan_kernel_us": round(scan_ms * 1000, 2),
                     "scan_kernel_frac": round(scan_bytes / (scan_ms * 1e-3) / 1e9 / hbm, 4)},
        "timing": {"value_source": graph_note or "eager launches", "eager_us": round(eager_ms * 1000, 2),
                   "graph_1_per_replay_us": round(per_replay_ms * 1000, 2) if per_replay_ms else None},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "throughput": {"value": round(P * n_total / (us * 1e-6) / 1e9, 2),
                       "unit": "G (token, head) codes scanned per s"},
    }
    if flushed_ms is not None:
        fa = alg_bytes / (flushed_ms * 1e-3) / 1e9
        line["value_l2_flushed"] = round(flushed_ms * 1000, 2)
        line["roofline"]["frac_l2_flushed"] = round(fa / hbm, 4)
    if sharded:
        line["sharded_decode"] = sharded
    if heads:
        line["head_sharded_decode"] = heads
    if decode:
        line["sparse_decode"] = decode
    if prefill:
        line["prefill_encode"] = prefill
    if decode4:
        line["batched_decode"] = decode4
    if accuracy:
        line["retrieval_accuracy"] = accuracy
    if train:
        line["hasher_training"] = train
    if config1:
        line["config1_decode"] = config1
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


def bench_prefill(torch, capi, ctx, dev, stream, args):
    """Config 4 prefill: K2 (tcgen05) encodes B=16 x 32 heads x 131072 bf16
    keys (17.2 GB) into 256-bit codes, one spl_encode_tc call per step.
    98,304 FLOP per key (2dh + 2hL)."""
    B, n, L4 = 16, 131072, 256
    rng = np.random.default_rng(4)
    w1 = (rng.standard_normal((H, D, D)) / np.sqrt(D)).astype(np.float32)
    b1 = np.zeros((H, D), np.float32)
    w2 = (rng.standard_normal((H, D, L4)) / np.sqrt(D)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    g = torch.Generator(device=dev)
    g.manual_seed(44)
    x = torch.empty((B, H, n, D), device=dev, dtype=torch.bfloat16)
    for b in range(B):  # fill in slices (keeps the f32 temporary small)
        x[b].copy_(torch.randn((H, n, D), generator=g, device=dev, dtype=torch.float32))
    codes = torch.empty((B, H, n, L4 // 32), device=dev, dtype=torch.int32)

    def step():
        hs.encode_tc(x, capi.SPL_BF16, B, n, codes, None, stream)

    for _ in range(args.warmup):
        step()
    steps = max(3, min(args.steps, 40))
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    time.sleep(0.3)
    l0 = ctx.launches()
    ms = event_timer(torch, step, steps, stream)
    launches = (ctx.launches() - l0) / steps
    clocks = clk.stop()
    keys = B * H * n
    flops = keys * (2 * D * D + 2 * D * L4)
    nbytes = keys * D * 2 + keys * (L4 // 32) * 4 + H * (D * D + D * L4) * 2
    burst, sustained, kind = tensor_peak()
    hbm, _ = peaks()
    tf = flops / (ms * 1e-3) / 1e12
    gbs = nbytes / (ms * 1e-3) / 1e9
    del x, codes
    hs.close() if hasattr(hs, "close") else None
    return {"workload": "config4 prefill: 16 x 32 heads x 131072 bf16 keys, d = h = 128, L = 256 "
                        "(K2 tcgen05, bf16 operands, fp32 TMEM accumulation)",
            "ms_per_step": round(ms, 3), "keys_per_s": round(keys / (ms * 1e-3) / 1e9, 3),
            "unit_keys": "G keys/s", "gpu_launches_per_step": launches,
            "clocks": clocks, "steps_timed": steps,
            # the leg runs `steps` x ~6 ms of back-to-back tensor work (power-
            # capped steady state), so its denominator is the sustained peak;
            # the burst fraction is kept beside it
            "roofline": {"tensor": {"achieved": round(tf, 1), "unit": "TFLOP/s", "peak": sustained,
                                    "peak_kind": f"{kind} sustained (kernel timed inside a long run)",
                                    "frac": round(tf / sustained, 4),
                                    "frac_of_burst": round(tf / burst, 4), "burst_peak": burst,
                                    "flops": flops},
                         "hbm": {"achieved": round(gbs, 1), "unit": "GB/s", "peak": hbm,
                                 "frac": round(gbs / hbm, 4), "algorithmic_bytes": nbytes}}}


def bench_decode4(torch, capi, ctx, dev, stream, args):
    """Config 4: B=16 sequences x 32 heads, 131072-token bf16 K/V caches,
    256-bit codes, k = 2% = 2621: one batched decode step (append each new
    key + value and its code, encode the queries, retrieve, sparse attend)."""
    B, n, L4 = 16, 131072, 256
    k = budget(n)
    P = B * H
    W4 = L4 // 32
    cap = n
    rng = np.random.default_rng(40)
    w1 = (rng.standard_normal((H, D, D)) / np.sqrt(D)).astype(np.float32)
    b1 = np.zeros((H, D), np.float32)
    w2 = (rng.standard_normal((H, D, L4)) / np.sqrt(D)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    codes = random_codes(torch, P, cap, W4, seed=56, dev=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(6)
    kc = torch.empty((B, H, cap, D), device=dev, dtype=torch.bfloat16)
    vc = torch.empty((B, H, cap, D), device=dev, dtype=torch.bfloat16)
    for b in range(B):
        kc[b].copy_(torch.randn((H, cap, D), generator=g, device=dev))
        vc[b].copy_(torch.randn((H, cap, D), generator=g, device=dev))
    q = torch.randn((B, H, D), generator=g, device=dev)
    kn = torch.randn((B, H, D), generator=g, device=dev)
    vn = torch.randn((B, H, D), generator=g, device=dev)
    nvalid = torch.full((B,), n, dtype=torch.int32, device=dev)
    idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros(P, dtype=torch.int32, device=dev)
    out = torch.zeros((B, H, D), dtype=torch.float32, device=dev)
    scale = float(1 / np.sqrt(D))

    def step(st=None):
        hs.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_BF16, cap, nvalid, n, k, scale,
                       idx, cnt, out, st if st is not None else stream)

    for _ in range(args.warmup):
        step()
    steps = min(args.steps, 20)
    l0 = ctx.launches()
    eager_ms = event_timer(torch, step, steps, stream)
    launches = (ctx.launches() - l0) / steps
    ctx.reserve(P, cap, L4, k, D)
    g_ms = graph_timer(torch, lambda st: step(st), steps, args.warmup)
    ms = g_ms if g_ms is not None else eager_ms

    qz = torch.randint(-2**31, 2**31 - 1, (P, W4), generator=g, device=dev, dtype=torch.int32)

    def retr():
        ctx.hamming_topk(codes, cap, L4, qz, P, nvalid, H, n, k, idx, cnt, stream)
    r_ms = event_timer(torch, retr, steps, stream)
    hbm, _ = peaks()
    alg = P * n * W4 * 4 + P * (k + 1) * D * 2 * 2 + H * (D * D + D + D * L4) * 4 + P * k * 4
    del kc, vc, codes
    return {"workload": "config4: B=16 x 32 heads, 131072-token bf16 K/V caches, 256-bit codes, "
                        "k=2621; append + encode + retrieve + attend",
            "us_per_step": round(ms * 1000, 2), "tok_per_s": round(B / (ms * 1e-3), 1),
            "timing": "CUDA graph replay of one decode step" if g_ms is not None else "eager",
            "eager_us_per_step": round(eager_ms * 1000, 2),
            "unit": "tok/s (one 32-head layer, 16 sequences)", "gpu_launches_per_step": launches,
            "retrieval_us": round(r_ms * 1000, 2),
            "roofline": {"bound": "hbm", "algorithmic_bytes": alg,
                         "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "peak": hbm,
                         "frac": round(alg / (ms * 1e-3) / 1e9 / hbm, 4)}}



def bench_train(capi, ctx, args):
    """Hasher training through the C-ABI (spl_train_hasher,
    host weights and data in, host weights and records out): the CLI's
    default training shape (spotlight.cpp:130-146: MLP d=h=L=128, max_oth 256,
    query subsample 64, maskout 0.98) on one synthetic 4096-token sequence.
    ms per iteration = (wall of a 64-iteration run - wall of a 1-iteration
    run) / 63, so the per-sequence preparation (exact logits, per-row order)
    and the holdout IoU cancel out. The reference's train_hasher runs the same
    workload on the host cores for a few iterations beside it, and the
    weights after those iterations are compared."""
    from oracle_lib import RefLib

    n, iters = 4096, 64
    rng = np.random.default_rng(0)
    data = [(rng.standard_normal((n, 128)).astype(np.float32),
             rng.standard_normal((n, 128)).astype(np.float32))]
    rank = dict(beta=1.0, alpha=3.0, maskout=0.98, max_top=None, max_oth=256,
                query_subsample=64)
    if not RefLib.available():
        return None
    ref = RefLib()
    w = ref.mlp_gaussian_init(128, 128, 128, 64.0, ref.derive_seed(0, 100))

    def gpu(it):
        g = [a.copy() for a in w]
        t = time.perf_counter()
        out = ctx.train_hasher(1, 128, 128, 128, 64.0, *g, data, capi.RankConfig(**rank),
                               capi.TrainConfig(num_iters=it))
        return time.perf_counter() - t, g, out["loop_ms"]

    gpu(2)
    runs = [gpu(iters) for _ in range(3)]
    ms_gpu = statistics.median(r[2] for r in runs) / iters
    e2e_s = statistics.median(r[0] for r in runs)
    ref_iters = 4
    cfg = dict(num_iters=1, warmup_iters=81, batch=1, seed=0, holdout_queries=128, max_lr=1e-3,
               min_lr=0.0, adam_beta1=0.9, adam_beta2=0.98, adam_eps=1e-8, weight_decay=0.1,
               grad_clip=1.0, soft_gamma=64.0, holdout_budget_rate=0.02)
    t = time.perf_counter()
    ref.train(1, *w, 64.0, data, rank, cfg)
    r1 = time.perf_counter() - t
    t = time.perf_counter()
    r = ref.train(1, *w, 64.0, data, rank, dict(cfg, num_iters=ref_iters))
    r4 = time.perf_counter() - t
    ms_ref = (r4 - r1) / (ref_iters - 1) * 1e3
    _, g4, _ = gpu(ref_iters)
    same = all(np.array_equal(a, b) for a, b in zip(g4, r[:3]))
    return {"workload": "train_hasher, MLP d=h=L=128, one 4096-token sequence, ranking loss, "
                        "max_oth 256, query subsample 64 (CLI defaults), AdamW",
            "ms_per_iter": round(ms_gpu, 3), "iters_timed": iters,
            "timing": "CUDA events around the iteration loop inside spl_train_hasher "
                      "(median of 3 runs)",
            "e2e_s_per_run": round(e2e_s, 4),
            "e2e_path": "spl_train_hasher wall time for %d iterations: host data and weights in, "
                        "exact logits + order, loop, weights and records out, holdout IoU" % iters,
            "reference_ms_per_iter": round(ms_ref, 3),
            "reference_threads": int(ref.lib.spotref_max_threads()),
            "speedup_vs_reference": round(ms_ref / ms_gpu, 1),
            "weights_identical_after_%d_iters" % ref_iters: bool(same)}


def bench_config1(torch, capi, ctx, dev, stream, args):
    """Config 1 (BASELINE configs[0]): one head, d=128, 4,096 cached f32 keys,
    128-bit MLP codes, k=64: one decode step (append the new key + encode the
    query + retrieve + sparse attention), latency (L2-resident), beside the
    reference's per-query path on the host (nxor_scores_into + top_k_indices +
    sparse_attention for the same query and cache)."""
    from oracle_lib import RefLib

    n, k, Hh = 4096, 64, 1
    rng = np.random.default_rng(41)
    w1 = (rng.standard_normal((Hh, D, D)) / np.sqrt(D)).astype(np.float32)
    b1 = np.zeros((Hh, D), np.float32)
    w2 = (rng.standard_normal((Hh, D, L)) / np.sqrt(D)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    W = L // 32
    keys = rng.standard_normal((n, D)).astype(np.float32)
    vals = rng.standard_normal((n, D)).astype(np.float32)
    qv = rng.standard_normal((1, D)).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    kc, vc = t(keys[None, None]), t(vals[None, None])
    codes = torch.zeros((1, 1, n, W), dtype=torch.int32, device=dev)
    hs.encode(t(keys[None, None]), 1, n, codes)  # exact codes of the cache
    q = t(qv[None])
    kn, vn = t(keys[None, None, n - 1]), t(vals[None, None, n - 1])
    nvalid = torch.full((1,), n, dtype=torch.int32, device=dev)
    idx = torch.zeros((1, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.zeros((1, 1, D), dtype=torch.float32, device=dev)
    scale = float(1 / np.sqrt(D))

    def step(st=None):
        hs.decode_step(q, kn, vn, 1, codes, kc, vc, capi.SPL_F32, n, nvalid, n, k, scale, idx, cnt,
                       out, st if st is not None else stream)

    for _ in range(args.warmup):
        step()
    eager_ms = event_timer(torch, step, args.steps, stream)
    ctx.reserve(1, n, L, k, D)
    g_ms = graph_timer(torch, lambda st: step(st), args.steps, args.warmup)
    ms = g_ms if g_ms is not None else eager_ms
    res = {"workload": "config1: 1 head, d=128, 4096 f32 keys, 128-bit codes, k=64; append + "
                       "encode + retrieve + sparse attend",
           "us_per_step": round(ms * 1000, 2), "eager_us_per_step": round(eager_ms * 1000, 2),
           "timing": "CUDA graph replay of one decode step" if g_ms is not None else "eager",
           "bound": "latency (L2-resident: 64 KB of codes, 65 x 1 KB K/V rows)"}
    if RefLib.available():
        ref = RefLib()
        c_np = codes.cpu().numpy().view(np.uint32).reshape(1, n, W)
        qc = np.zeros((1, W), np.uint32)
        qcode = torch.zeros((1, 1, 1, W), dtype=torch.int32, device=dev)
        hs.encode(q[None], 1, 1, qcode)
        qc[0] = qcode.cpu().numpy().view(np.uint32).reshape(-1)
        h = ref.index_create(c_np, np.array([n], np.uint32))
        try:
            times = []
            for i in range(25):
                t0 = time.perf_counter()
                sel = ref.retrieve_batch(h, qc, np.array([n], np.uint32), k, threads=1)
                picked = sorted(set(sel[0].tolist()) | {n - 1})
                ref.sparse_attention(qv, keys, vals, scale, np.array([n], np.uint32), [picked])
                if i >= 5:
                    times.append((time.perf_counter() - t0) * 1e6)
        finally:
            ref.index_destroy(h)
        res["reference_us_per_step"] = round(statistics.median(times), 1)
        res["reference_path"] = ("unmodified reference: nxor_scores_into + top_k_indices + "
                                 "sparse_attention, one host thread (the encode of the query "
                                 "excluded on the reference side)")
        same = sorted(idx[0, :int(cnt[0])].cpu().numpy().view(np.uint32).tolist()) == sorted(sel[0].tolist())
        res["indices_equal_reference"] = bool(same)
    return res

def bench_accuracy(torch, capi, ctx, dev, stream, args):
    """Retrieval accuracy (the paper's Table-1 metric) at the
    config-2 shape: IoU of the MLP-hash top-k (exact codes of the actual
    keys, K3) with the exact dense top-k (spl_oracle_topk), per head, plus
    the dense oracle's own time. Random-init hasher on Gaussian keys, so the
    IoU is the untrained baseline; trained SPLH checkpoints raise it."""
    Hh, n, d, L2 = 32, 131072, 128, 128
    k = budget(n)
    rng = np.random.default_rng(21)
    w1 = (rng.standard_normal((Hh, d, d)) / np.sqrt(d)).astype(np.float32)
    b1 = np.zeros((Hh, d), np.float32)
    w2 = (rng.standard_normal((Hh, d, L2)) / np.sqrt(d)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    g = torch.Generator(device=dev)
    g.manual_seed(21)
    keys = torch.randn((1, Hh, n, d), generator=g, device=dev, dtype=torch.float32)
    q = torch.randn((1, Hh, d), generator=g, device=dev, dtype=torch.float32)
    codes = torch.empty((1, Hh, n, L2 // 32), device=dev, dtype=torch.int32)
    hs.encode(keys, 1, n, codes, capi.SPL_ENCODE_EXACT, stream)
    qc = torch.empty((1, Hh, L2 // 32), device=dev, dtype=torch.int32)
    hs.encode(q, 1, 1, qc, capi.SPL_ENCODE_EXACT, stream)
    nv = torch.full((1,), n, dtype=torch.int32, device=dev)
    hidx = torch.zeros((Hh, k), dtype=torch.int32, device=dev)
    hcnt = torch.zeros(Hh, dtype=torch.int32, device=dev)
    ctx.hamming_topk(codes, n, L2, qc, Hh, nv, Hh, n, k, hidx, hcnt, stream)
    oidx = torch.zeros((Hh, k), dtype=torch.int32, device=dev)
    ocnt = torch.zeros(Hh, dtype=torch.int32, device=dev)
    scale = float(1 / np.sqrt(d))

    def oracle():
        ctx.oracle_topk(q[0], keys, capi.SPL_F32, n, d, Hh, nv, Hh, n, scale, k, oidx, ocnt,
                        None, stream)
    oracle()
    o_ms = event_timer(torch, oracle, 5, stream)
    out = torch.zeros(Hh, dtype=torch.float64, device=dev)
    ctx.iou(hidx, hcnt, k, oidx, ocnt, k, Hh, out, stream)
    # K2 fast-mode drift (BASELINE parity contract): the same retrieval from
    # the tcgen05 encoder's codes (bf16 operands) of the same keys — IoU with
    # the dense oracle, and with the exact (K1) hash top-k
    codes2 = torch.empty_like(codes)
    hs.encode_tc(keys, capi.SPL_F32, 1, n, codes2, None, stream)
    t_idx = torch.zeros((Hh, k), dtype=torch.int32, device=dev)
    t_cnt = torch.zeros(Hh, dtype=torch.int32, device=dev)
    ctx.hamming_topk(codes2, n, L2, qc, Hh, nv, Hh, n, k, t_idx, t_cnt, stream)
    out_tc = torch.zeros(Hh, dtype=torch.float64, device=dev)
    ctx.iou(t_idx, t_cnt, k, oidx, ocnt, k, Hh, out_tc, stream)
    out_x = torch.zeros(Hh, dtype=torch.float64, device=dev)
    ctx.iou(t_idx, t_cnt, k, hidx, hcnt, k, Hh, out_x, stream)
    torch.cuda.synchronize()
    diff_bits = int(np.unpackbits(torch.bitwise_xor(codes, codes2).cpu().numpy().view(np.uint8)).sum())
    ious = out.cpu().numpy()
    ious_tc, ious_x = out_tc.cpu().numpy(), out_x.cpu().numpy()
    del keys, codes, codes2
    return {"workload": "config2 shape: 32 heads x 131072 f32 keys, d=128, 128-bit exact MLP codes, "
                        "k=2621; IoU(hash top-k, exact dense top-k) per head",
            "mean_iou": round(float(ious.mean()), 4), "min_iou": round(float(ious.min()), 4),
            "max_iou": round(float(ious.max()), 4),
            "oracle_topk_us": round(o_ms * 1000, 1),
            "k2_fast_mode": {"mean_iou_vs_oracle": round(float(ious_tc.mean()), 4),
                             "mean_iou_vs_exact_hash_topk": round(float(ious_x.mean()), 4),
                             "min_iou_vs_exact_hash_topk": round(float(ious_x.min()), 4),
                             "code_bits_differing_from_exact": diff_bits,
                             "code_bits_total": int(Hh * n * L2),
                             "note": "keys encoded by K2 (tcgen05, bf16 operands, fp32 accumulation) "
                                     "instead of K1 (bit-exact); the query code is exact in both"},
            "data": "synthetic Gaussian keys/queries, random-init hasher (untrained baseline)"}


def bench_decode(torch, capi, ctx, dev, stream, args, hasher_c3):
    """Config 2: B=1, 32 heads, 128K context, k=2% = 2621, bf16 K/V; one full
    decode step (append new key + encode query + retrieve + sparse attend)."""
    B, n = 1, 131072
    k = budget(n)
    P = B * H
    W = L // 32
    cap = n
    codes = random_codes(torch, P, cap, W, seed=55, dev=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    kc = torch.randn((B, H, cap, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    vc = torch.randn((B, H, cap, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    q = torch.randn((B, H, D), generator=g, device=dev)
    kn = torch.randn((B, H, D), generator=g, device=dev)
    vn = torch.randn((B, H, D), generator=g, device=dev)
    nvalid = torch.full((B,), n, dtype=torch.int32, device=dev)
    idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros(P, dtype=torch.int32, device=dev)
    out = torch.zeros((B, H, D), dtype=torch.float32, device=dev)
    scale = float(1 / np.sqrt(D))

    def step(st=None):
        hasher_c3.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_BF16, cap, nvalid, n, k, scale,
                              idx, cnt, out, st if st is not None else stream)

    for _ in range(args.warmup):
        step()
    l0 = ctx.launches()
    ctx.launch_log()
    eager_ms = event_timer(torch, step, args.steps, stream)
    launches = ctx.launches() - l0
    kernels = ctx.launch_log()[: launches // args.steps]
    ctx.reserve(P, cap, L, k, D)
    # the step's working set (67 MB of codes + 43 MB of gathered K/V rows) fits
    # the 126 MB L2, so it is timed with L2 flushed before every step: the
    # device time per step from CUDA graphs of steps x (flush, step) minus
    # steps x flush, and (second number) the median of CUDA events around
    # single graph replays, which also holds the replay's launch gap
    g_warm = graph_timer(torch, lambda st: step(st), args.steps, args.warmup)
    fl = flushed_graph_timer(torch, lambda st: step(st), min(args.steps, 20), args.warmup)
    g_ms = graph_timer(torch, lambda st: step(st), args.steps, args.warmup, flush=True)
    ms = fl[0] if fl else (g_ms if g_ms is not None else eager_ms)
    def att():  # K4 alone over the same lists (the two-launch form of the step)
        ctx.sparse_attend(q, kc, vc, capi.SPL_BF16, cap, D, P, idx, k, cnt, nvalid, H, scale, out, stream)
    att_ms = flushed_timer(torch, att, args.steps, stream)
    hbm, _ = peaks()
    alg = P * n * W * 4 + P * (k + 1) * D * 2 * 2 + H * (D * D + D + D * L) * 4 + P * k * 4
    return {"workload": "config2: B=1, 32 heads, 131072-token bf16 K/V cache, 128-bit codes, k=2621",
            "us_per_step": round(ms * 1000, 2), "tok_per_s": round(B / (ms * 1e-3), 1),
            "timing": ("device time per step, L2 flushed before each: CUDA graphs of steps x "
                       "(flush, step) minus steps x flush" if fl else "eager"),
            "us_per_step_events": round(g_ms * 1000, 2) if g_ms is not None else None,
            "us_per_step_events_note": "median of CUDA events around one graph replay each, L2 "
                                       "flushed before each (includes the replay launch gap)",
            "us_per_step_l2_warm": round(g_warm * 1000, 2) if g_warm is not None else None,
            "eager_us_per_step": round(eager_ms * 1000, 2),
            "unit": "tok/s (one 32-head layer)", "gpu_launches_per_step": launches / args.steps,
            "kernels_per_step": kernels,
            "k4_standalone_attend_us": round(att_ms * 1000, 2),
            "roofline": {"bound": "hbm", "algorithmic_bytes": alg,
                         "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "peak": hbm,
                         "frac": round(alg / (ms * 1e-3) / 1e9 / hbm, 4)}}



def bench_sharded_decode(torch, capi, ctx, dev, stream, args, world, rank, dist, same_gpu,
                         all_reduce_dev):
    """Config 5: one decode step of a 32-head layer over a sequence-sharded KV
    cache — 512K tokens per GPU (weak scaling: N x 512K in total), 128-bit
    codes, bf16 K/V, k = 2% of the whole cache — through
    spl_sharded_decode_step on every rank: encode (the last rank appends the
    new token), retrieval with the in-kernel histogram exchange, partial
    attention, in-kernel exchange of the (m, l, o) partials, combine. At
    N = 1 the same call runs with a 1-rank group (the point the scaling curve
    starts from). tok/s = 1 / step (one sequence)."""
    n = N_TOK
    n_total = n * world
    k = budget(n_total)
    P = H
    W = L // 32
    rng = np.random.default_rng(50)
    w1 = (rng.standard_normal((H, D, D)) / np.sqrt(D)).astype(np.float32)
    b1 = np.zeros((H, D), np.float32)
    w2 = (rng.standard_normal((H, D, L)) / np.sqrt(D)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    codes = random_codes(torch, P, n, W, seed=500 + rank, dev=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(600 + rank)
    kc = torch.empty((1, H, n, D), device=dev, dtype=torch.bfloat16)
    vc = torch.empty((1, H, n, D), device=dev, dtype=torch.bfloat16)
    for h0 in range(0, H, 8):
        kc[0, h0:h0 + 8].copy_(torch.randn((8, n, D), generator=g, device=dev))
        vc[0, h0:h0 + 8].copy_(torch.randn((8, n, D), generator=g, device=dev))
    gq = torch.Generator(device=dev)
    gq.manual_seed(7)  # the step's inputs are the same on every rank
    q = torch.randn((1, H, D), generator=gq, device=dev)
    kn = torch.randn((1, H, D), generator=gq, device=dev)
    vn = torch.randn((1, H, D), generator=gq, device=dev)
    nvalid = torch.full((1,), n, dtype=torch.int32, device=dev)
    idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros(P, dtype=torch.int32, device=dev)
    off = torch.zeros(P, dtype=torch.int32, device=dev)
    out = torch.zeros((1, H, D), dtype=torch.float32, device=dev)
    scale = float(1 / np.sqrt(D))
    owner = rank == world - 1

    def agree(ok):
        """All ranks leave together: a failure on any rank (peer mapping,
        device error) ends the leg on every rank instead of leaving the others
        inside a collective."""
        if not dist:
            return ok
        t = torch.tensor([1 if ok else 0], device=dev)
        all_reduce_dev(t, dist.ReduceOp.MIN)
        return int(t.item()) == 1

    peer, err = None, None
    try:
        peer = ctx.peer(world, rank, P, L)
        if world == 1:
            capi.Peer.connect_local(ctx, [peer])
        else:
            handles = [None] * world
            dist.all_gather_object(handles, peer.ipc_handle())
            if os.environ.get("SPL_BENCH_FAIL_PEER_RANK") == str(rank):  # test hook: one-sided failure
                raise RuntimeError("injected peer-open failure")
            peer.open(handles)
        ctx.reserve(P, n, L, k, D)
    except Exception as e:  # e.g. no CUDA IPC / peer access between these GPUs
        err = f"peer setup: {str(e)[:120]}"
    if not agree(err is None):
        if peer is not None:
            peer.close()
        return {"workload": f"config5 over {world} GPU(s)", "error": err or "peer setup failed on another rank"}
    # the step appends at n_valid - 1: keep the cache length fixed across the
    # timed steps (each step rewrites the same slot), as a decode loop at a
    # fixed context would

    def step(st=None):
        hs.sharded_decode_step(peer, q, kn, vn, 1, owner, codes, kc, vc, capi.SPL_BF16, n, nvalid, n,
                               k, scale, idx, cnt, off, out, st if st is not None else stream)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    ctx.launch_log()
    try:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        ctx.check_device_error()
    except Exception as e:
        err = f"sharded step: {str(e)[:120]}"
    if not agree(err is None):
        peer.close()
        return {"workload": f"config5 over {world} GPU(s)", "error": err or "sharded step failed on another rank"}
    barrier()
    kernels = ctx.launch_log()
    launches = len(kernels) / max(1, args.warmup)
    steps = min(args.steps, 20)
    barrier()
    eager_ms = event_timer(torch, step, steps, stream)
    barrier()
    fl = flushed_graph_timer(torch, lambda st: step(st), steps, args.warmup) if not same_gpu else None
    barrier()
    ctx.check_device_error()
    ms = fl[0] if fl else eager_ms
    # e2e through the C-ABI with host buffers: H2D of the step's q / k_new /
    # v_new, the sharded step, D2H of the attention output
    qh, knh, vnh = (t.cpu().pin_memory() for t in (q, kn, vn))
    outh = torch.empty_like(out, device="cpu").pin_memory()

    def e2e_step():
        q.copy_(qh, non_blocking=True)
        kn.copy_(knh, non_blocking=True)
        vn.copy_(vnh, non_blocking=True)
        step()
        outh.copy_(out, non_blocking=True)
    for _ in range(3):
        e2e_step()
    barrier()
    e2e_ms = event_timer(torch, e2e_step, steps, stream)
    barrier()
    t = torch.tensor([ms, eager_ms, e2e_ms], device=dev)
    if dist:
        all_reduce_dev(t, dist.ReduceOp.MAX)
    ms, eager_ms, e2e_ms = (float(x) for x in t.tolist())
    hbm, _ = peaks()
    # algorithmic bytes per rank: codes + this rank's
    # share of the gathered K/V rows (k/N on average) + weights + indices +
    # the exchanged histograms and partials
    alg = (P * n * W * 4 + P * (k // world + 1) * D * 2 * 2 + H * (D * D + D + D * L) * 4
           + P * (k // world) * 4 + world * P * ((L + 2) + (D + 2)) * 8)
    peer.close()
    del kc, vc, codes
    torch.cuda.empty_cache()
    return {"workload": f"config5: one sequence, {n_total} tokens sequence-sharded over {world} GPU(s) "
                        f"({n} per GPU), 32 heads, d=128, bf16 K/V, 128-bit codes, k={k}; encode + "
                        "append (last rank) + retrieval + partial attention + combine",
            "us_per_step": round(ms * 1000, 2), "tok_per_s": round(1.0 / (ms * 1e-3), 1),
            "unit": "tok/s (one 32-head layer, one sequence; max over ranks)",
            "timing": ("device time per step with L2 flushed before each, from CUDA graphs of "
                       "steps x (flush, step) minus steps x flush" if fl else "eager launches"),
            "eager_us_per_step": round(eager_ms * 1000, 2),
            "e2e": {"value": round(1.0 / (e2e_ms * 1e-3), 1), "unit": "tok/s",
                    "us_per_step": round(e2e_ms * 1000, 2),
                    "h2d_bytes_per_step": 3 * H * D * 4, "d2h_bytes_per_step": H * D * 4,
                    "path": "spl_sharded_decode_step with pinned host q / k_new / v_new in and the "
                            "attention output out, every rank"},
            "kernels_per_step": kernels[: int(launches)], "gpu_launches_per_step": launches,
            "exchange": ("in-kernel over IPC-mapped peer memory (NVLink between GPUs): per-head "
                         "score histograms, then the (m, l, o) attention partials"),
            "roofline": {"bound": "hbm", "algorithmic_bytes_per_rank": alg,
                         "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "peak": hbm,
                         "frac": round(alg / (ms * 1e-3) / 1e9 / hbm, 4)}}


def bench_head_sharded(torch, capi, ctx, dev, stream, args, world, rank, dist, same_gpu,
                       all_reduce_dev):
    """Head sharding (SURVEY §8 e): the same config-5 cache split by heads
    instead — every rank holds all N x 512K tokens of 32 / N heads (equal
    bytes per rank to the sequence split) and runs the unsharded decode step
    on them; heads are independent (one hasher per head), so there is no
    exchange and the output stays head-sharded."""
    if H % world:
        return None
    Hr = H // world
    n = N_TOK * world
    k = budget(n)
    W = L // 32
    rng = np.random.default_rng(51 + rank)
    w1 = (rng.standard_normal((Hr, D, D)) / np.sqrt(D)).astype(np.float32)
    b1 = np.zeros((Hr, D), np.float32)
    w2 = (rng.standard_normal((Hr, D, L)) / np.sqrt(D)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    codes = random_codes(torch, Hr, n, W, seed=700 + rank, dev=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(800 + rank)
    kc = torch.empty((1, Hr, n, D), device=dev, dtype=torch.bfloat16)
    vc = torch.empty((1, Hr, n, D), device=dev, dtype=torch.bfloat16)
    for h in range(Hr):
        kc[0, h].copy_(torch.randn((n, D), generator=g, device=dev))
        vc[0, h].copy_(torch.randn((n, D), generator=g, device=dev))
    q = torch.randn((1, Hr, D), generator=g, device=dev)
    kn = torch.randn((1, Hr, D), generator=g, device=dev)
    vn = torch.randn((1, Hr, D), generator=g, device=dev)
    nvalid = torch.full((1,), n, dtype=torch.int32, device=dev)
    idx = torch.zeros((Hr, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros(Hr, dtype=torch.int32, device=dev)
    out = torch.zeros((1, Hr, D), dtype=torch.float32, device=dev)
    scale = float(1 / np.sqrt(D))
    ctx.reserve(Hr, n, L, k, D)

    def step(st=None):
        hs.decode_step(q, kn, vn, 1, codes, kc, vc, capi.SPL_BF16, n, nvalid, n, k, scale, idx, cnt,
                       out, st if st is not None else stream)
    ctx.launch_log()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    kernels = ctx.launch_log()
    steps = min(args.steps, 20)
    if dist:
        dist.barrier()
    fl = flushed_graph_timer(torch, lambda st: step(st), steps, args.warmup) if not same_gpu else None
    ms = fl[0] if fl else event_timer(torch, step, steps, stream)
    t = torch.tensor([ms], device=dev)
    if dist:
        all_reduce_dev(t, dist.ReduceOp.MAX)
    ms = float(t.item())
    del kc, vc, codes
    torch.cuda.empty_cache()
    return {"workload": f"config5 by heads: {n} tokens x {Hr} heads per GPU ({world} GPUs x {Hr} = 32 "
                        f"heads), bf16 K/V, 128-bit codes, k={k}; no exchange",
            "us_per_step": round(ms * 1000, 2), "tok_per_s": round(1.0 / (ms * 1e-3), 1),
            "unit": "tok/s (one 32-head layer, one sequence; max over ranks)",
            "timing": ("device time per step with L2 flushed before each (graph difference)" if fl
                       else "eager launches"),
            "kernels_per_step": kernels[: len(kernels) // max(1, args.warmup)]}


if __name__ == "__main__":
    main()
