"""Where does the e2e step time go? (measurement aid, not a bench line)
Config-3 retrieval with the query H2D + exact encode + retrieval + indices
D2H, as one CUDA graph per step: variants without the D2H, with the D2H
serial, and with the previous step's D2H on a parallel branch."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_19740_b200 import capi  # noqa: E402

P, n, L, D = 32, 524288, 128, 128
k = capi.budget_from_rate(0.02, n)
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
rng = np.random.default_rng(7)
w1 = (rng.standard_normal((P, D, D)) / np.sqrt(D)).astype(np.float32)
b1 = np.zeros((P, D), np.float32)
w2 = (rng.standard_normal((P, D, L)) / np.sqrt(D)).astype(np.float32)
hs = ctx.hasher(w1, b1, w2)
g = torch.Generator(device=dev)
g.manual_seed(5)
codes = torch.randint(-2**31, 2**31 - 1, (P, n, L // 32), generator=g, device=dev, dtype=torch.int32)
nv = torch.full((P,), n, dtype=torch.int32, device=dev)
qc = torch.zeros((1, P, L // 32), dtype=torch.int32, device=dev)
q_host = torch.randn((1, P, D)).pin_memory()
q_dev = torch.empty((1, P, D), device=dev)
idx = [torch.zeros((P, k), dtype=torch.int32, device=dev) for _ in range(2)]
cnt = [torch.zeros(P, dtype=torch.int32, device=dev) for _ in range(2)]
idx_h = [torch.empty((P, k), dtype=torch.int32).pin_memory() for _ in range(2)]
cnt_h = [torch.empty(P, dtype=torch.int32).pin_memory() for _ in range(2)]
gs, cps = torch.cuda.Stream(), torch.cuda.Stream()
ctx.reserve(P, n, L, k, D)
compute(0, torch.cuda.current_stream()) if False else None


def compute(b, st):
    q_dev.copy_(q_host, non_blocking=True)
    hs.encode(q_dev, 1, 1, qc, capi.SPL_ENCODE_EXACT, st)
    ctx.hamming_topk(codes, n, L, qc, P, nv, 1, n, k, idx[b], cnt[b], st)


ctx.hamming_topk(codes, n, L, qc, P, nv, 1, n, k, idx[0], cnt[0])
torch.cuda.synchronize()


def d2h(b):
    idx_h[b].copy_(idx[b], non_blocking=True)
    cnt_h[b].copy_(cnt[b], non_blocking=True)


def capture(body):
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=gs, capture_error_mode="relaxed"):
        body()
    return gr


def timeit(graphs, steps=50, tail=None):
    for i in range(4):
        graphs[i % len(graphs)].replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            graphs[i % len(graphs)].replay()
        if tail:
            tail()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1000 / steps)
    return best


def par(b):
    def body():
        fork = torch.cuda.Event()
        fork.record(gs)
        cps.wait_event(fork)
        with torch.cuda.stream(cps):
            d2h(1 - b)
        compute(b, gs)
        join = torch.cuda.Event()
        join.record(cps)
        gs.wait_event(join)
    return body


print(f"retrieval only (q codes 0) {timeit([capture(lambda: ctx.hamming_topk(codes, n, L, qc, P, nv, 1, n, k, idx[0], cnt[0], gs))]):7.2f} us")
hs.encode(q_dev.copy_(q_host), 1, 1, qc, capi.SPL_ENCODE_EXACT)
torch.cuda.synchronize()
print("q codes now", qc.view(-1)[:4].tolist())
print(f"retrieval only (encoded q) {timeit([capture(lambda: ctx.hamming_topk(codes, n, L, qc, P, nv, 1, n, k, idx[0], cnt[0], gs))]):7.2f} us")
print(f"H2D + encode + retrieval {timeit([capture(lambda: compute(0, gs))]):7.2f} us")
print(f"D2H only                 {timeit([capture(lambda: d2h(0))]):7.2f} us")
print(f"serial (with D2H)        {timeit([capture(lambda: (compute(0, gs), d2h(0)))]):7.2f} us")
print(f"pipelined (prev D2H par) {timeit([capture(par(0)), capture(par(1))], tail=lambda: d2h(1)):7.2f} us")



# variant: compute graphs on one stream, the D2H as plain async copies on a
# second stream ordered by events (single-branch graphs)
cg = [capture(lambda: compute(0, gs)), capture(lambda: compute(1, gs))]
enc_g = capture(lambda: hs.encode(q_dev, 1, 1, qc, capi.SPL_ENCODE_EXACT, gs))
h2d_g = capture(lambda: q_dev.copy_(q_host, non_blocking=True))
print(f"encode only              {timeit([enc_g]):7.2f} us")
print(f"H2D only                 {timeit([h2d_g]):7.2f} us")


def two_stream(steps=50):
    cur = torch.cuda.current_stream()
    done = [None, None]
    for _ in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for i in range(steps):
            b = i & 1
            if done[b] is not None:
                cur.wait_event(done[b])
            cg[b].replay()
            r = torch.cuda.Event()
            r.record(cur)
            cps.wait_event(r)
            with torch.cuda.stream(cps):
                d2h(b)
            d = torch.cuda.Event()
            d.record(cps)
            done[b] = d
        for d in done:
            cur.wait_event(d)
        e1.record(cur)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / steps


print(f"pipelined (2 streams)    {two_stream():7.2f} us")


# variant: graph i = retrieval(i) ‖ [D2H(i-1)] ‖ [H2D(i+1) -> encode(i+1)]
# (double-buffered query vectors / codes / indices): the next query's encode
# runs on the SMs the retrieval's last CTAs leave free
qd = [torch.empty((1, P, D), device=dev) for _ in range(2)]
qcs = [torch.zeros((1, P, L // 32), dtype=torch.int32, device=dev) for _ in range(2)]
cs2 = torch.cuda.Stream()


def pipe3(b):
    def body():
        fork = torch.cuda.Event()
        fork.record(gs)
        cps.wait_event(fork)
        cs2.wait_event(fork)
        with torch.cuda.stream(cps):
            d2h(1 - b)
        with torch.cuda.stream(cs2):
            qd[1 - b].copy_(q_host, non_blocking=True)
            hs.encode(qd[1 - b], 1, 1, qcs[1 - b], capi.SPL_ENCODE_EXACT, cs2)
        ctx.hamming_topk(codes, n, L, qcs[b], P, nv, 1, n, k, idx[b], cnt[b], gs)
        j1, j2 = torch.cuda.Event(), torch.cuda.Event()
        j1.record(cps)
        j2.record(cs2)
        gs.wait_event(j1)
        gs.wait_event(j2)
    return body


def prologue():
    qd[0].copy_(q_host, non_blocking=True)
    hs.encode(qd[0], 1, 1, qcs[0], capi.SPL_ENCODE_EXACT)


prologue()
torch.cuda.synchronize()
p3 = [capture(pipe3(0)), capture(pipe3(1))]
print(f"pipelined (D2H and next encode in parallel) {timeit(p3, tail=lambda: d2h(1)):7.2f} us")
