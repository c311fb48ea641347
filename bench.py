#!/usr/bin/env python
"""LDBP hot-path benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch:
forward, waveform-MSE seed, backward, fp64 reductions, all-reduce (N > 1) and Adam — the C3
"LDBP training step" of BASELINE.json (512 blocks x 2^14 samples, M = 50, T = 9, gamma'
learnable) on every rank (weak scaling: per-GPU work fixed).  `value` is the whole-job
throughput in Gsample*steps/s = (sum over ranks of B*n) * M / step time / 1e9.  The forward-only
configurations (C2, C4) and the 2^28-sample training configuration (C5) are reported under
"extra" on single-GPU runs.

Inputs are synthetic and seeded (ldbp_inputs): band-limited circular Gaussian blocks with per-
block launch power drawn from P = {-2,-1,0,1} dBm, LS inverse-CD taps (gain-capped) and the DBP
gamma' schedule.  L2 is flushed (a 256 MiB write) between timed steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LDBP Gsample·steps/s fwd and fwd+bwd at 1/2/4/8 B200; % of FP32/HBM roofline"
UNIT = "Gsample·steps/s"
POWERS_DBM = (-2.0, -1.0, 0.0, 1.0)  # training power set of §V-A

CONFIGS = {
    # name: blocks (per GPU when weak-scaled, global when strong-scaled), samples per block, spans,
    # steps per span, taps, mode, seed index (ldbp_inputs keyed streams), default scaling (BJ configs:
    # C4 "2^26 total samples sharded across 1/2/4/8 GPUs" and C5 "8192 blocks on 8 GPUs" fix the
    # global batch; C1-C3 fix the per-GPU batch)
    "C1": dict(B=4, n=1024, spans=2, sps=2, T=3, mode="train", idx=1, scaling="weak"),
    "C2": dict(B=256, n=16384, spans=25, sps=1, T=5, mode="fwd", idx=2, scaling="weak"),
    "C3": dict(B=512, n=16384, spans=25, sps=2, T=9, mode="train", idx=3, scaling="weak"),
    "C4": dict(B=4096, n=16384, spans=25, sps=4, T=15, mode="fwd", idx=4, scaling="strong"),
    "C5": dict(B=8192, n=32768, spans=25, sps=1, T=3, mode="train", idx=5, scaling="strong"),
}
WORKLOAD = {
    "C1": "Tiny LDBP fwd+bwd: 4 blocks x 1024, M=4, T=3",
    "C2": "Long-haul LDBP inference: 256 blocks x 2^14, M=25 (1 StPS), T=5",
    "C3": "LDBP training step: 512 blocks x 2^14, M=50 (2 StPS), T=9, gamma' learnable, MSE vs tx waveform, fwd+bwd+Adam",
    "C4": "Unpruned-filter LDBP inference: 4096 blocks x 2^14, M=100 (4 StPS), T=15",
    "C5": "Data-parallel LDBP training: 8192 blocks x 2^15, M=25, T=3, gamma' learnable, fwd+bwd+allreduce+Adam",
}
SMS = 148
FP32_LANES_PER_SM = 128  # B200: 4 SMSPs x 32 FP32 lanes (B200_PROFILING.md / B300_MICROARCH.md)
L2_FLUSH_BYTES = 256 << 20


def instr_fwd(kh):
    """Algorithmic FP32 instructions per sample-step, forward (folded FIR 6Kh+4 + Kerr 8; §8(d))."""
    return 6 * kh + 12


def instr_bwd(kh):
    """Algorithmic FP32 instructions per sample-step of the reverse sweep (12Kh+18; §8(a) a6)."""
    return 12 * kh + 18


# ----------------------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi sampler (B200_PROFILING.md clocks line), started before the timed region."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(gpu_index)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, t0, t1):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        rows = []
        for line in open(self.path):
            p = [c.strip() for c in line.split(",")]
            if len(p) < 9:
                continue
            try:
                ts = time.mktime(time.strptime(p[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                rows.append((ts, float(p[2]), float(p[3]), p[5:9]))
            except ValueError:
                continue
        inwin = [r for r in rows if t0 - 1.0 <= r[0] <= t1 + 1.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inwin for i, v in enumerate(r[3]) if v.lower() == "active"})
        if not inwin:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(r[1] for r in inwin), "sm_max_mhz": max(r[2] for r in inwin),
                "reasons": reasons, "samples": len(inwin)}


# ----------------------------------------------------------------------------------------
# workload
# ----------------------------------------------------------------------------------------
def make_model(cfg):
    """Product-side model init (GPU leg): DBP step plan + gamma' (G3/G4) and LS inverse-CD taps
    with gain cap (G12b) from the package's host helpers."""
    import numpy as np

    from paper_2010_14258_b200 import init

    deltas, gamma = init.dbp_schedule(cfg["spans"], 80.0, cfg["sps"])
    taps = init.model_taps(deltas, cfg["T"], cap=1.0)
    return taps.astype(np.complex128), gamma


def make_model_oracle(cfg):
    """The same model from the oracle's own helpers (CPU legs: the reference arm and cpu_baseline
    never import the product package, so libldbp.so is never loaded into the oracle process)."""
    from oracle import physics, steps

    deltas, gamma = steps.dbp_plan(cfg["spans"], 80.0, cfg["sps"], 0.2, 1.3)
    taps = [steps.ls_taps(steps.xi_of(d, physics.ps2_per_km(-21.7), 21.4e9), cfg["T"], cap=1.0) for d in deltas]
    import numpy as np

    return np.stack(taps), gamma


def global_blocks(cfg, world, scaling):
    return cfg["B"] * world if scaling == "weak" else cfg["B"]


def my_blocks(cfg, world, rank, scaling):
    """Global block indices of this rank: contiguous shard (dp.shard) of the global batch."""
    from paper_2010_14258_b200.dp import shard

    return shard(rank, world, global_blocks(cfg, world, scaling))


def make_inputs(cfg, blocks, world=1, scaling="weak"):
    """Received blocks and tx targets keyed by GLOBAL block index (same union for any G): the GPU
    SSFM link (paper_2010_14258_b200.channel: 25 x 80 km, 16-QAM 10.7 GBd, rho_a = 4, EDFA ASE drawn
    in-kernel, LPF + decimation to 2 sps) on a pool of unique blocks, shifted / rotated per block."""
    from paper_2010_14258_b200 import channel

    blocks = list(blocks)
    nglob = global_blocks(cfg, world, scaling)
    U = min(256, max(4, 4 * -(-nglob // 4)))
    pool = channel.simulate_pool(cfg["idx"], U, cfg["n"] // channel.RHO_D)
    x, tgt = channel.link_blocks(cfg["idx"], blocks, cfg["n"], pool=pool)
    del pool
    return x, (tgt if cfg["mode"] == "train" else None)


def run_config(name, cfg, steps, warmup, world, rank, dev, want_e2e=True, want_clocks=True, scaling=None,
               force_collective=False):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2010_14258_b200 as P
    from paper_2010_14258_b200 import _lib
    from paper_2010_14258_b200.dp import DataParallelLDBP

    taps, gamma = make_model(cfg)
    M, T = taps.shape
    kh = (T - 1) // 2
    scaling = scaling or cfg["scaling"]
    blocks = my_blocks(cfg, world, rank, scaling)
    B, n = len(blocks), cfg["n"]
    x, tgt = make_inputs(cfg, blocks, world, scaling)
    train = cfg["mode"] == "train"
    st = P.TrainState.create(taps, gamma, device=dev)
    ws = P.Workspace()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    y = torch.empty_like(x)
    trainer = None
    if train:
        trainer = DataParallelLDBP(state=st, loss_grad_fn=lambda a, b: P.ldbp_loss_grad(a, b, st.taps, st.gamma, ws=ws),
                                   train_step_fn=lambda a, b: P.ldbp_train_step(st, a, b, ws=ws),
                                   force_collective=force_collective)
        trainer.set_local_samples(B * n)

    def step(xx, tt):
        if train:
            return trainer.step(xx, tt)
        return P.ldbp_forward(xx, st.taps, st.gamma, out=y, ws=ws)

    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        step(x, tgt)
    torch.cuda.synchronize()

    clocks = Clocks(torch.cuda.current_device()) if (want_clocks and rank == 0) else None
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(float(i))  # evict L2 between timed steps (outside the events)
        evs[i][0].record(stream)
        step(x, tgt)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    t_wall1 = time.time()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if dist.is_initialized():
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop(t_wall0, t_wall1) if clocks else None
    ms_per_step = ms / steps
    samples_global = global_blocks(cfg, world, scaling) * n
    value = samples_global * M / (ms_per_step * 1e-3) / 1e9

    # per-kernel durations, live (CUDA events around each launch, same stream), separate pass
    with P.api.trace(capacity=8192) as tr:
        for i in range(steps):
            flush.fill_(float(i))
            step(x, tgt)
        torch.cuda.synchronize()
    per_kind = {}
    for kind, nsteps, samples, kms in tr.records:
        d = per_kind.setdefault(kind, {"ms": 0.0, "launches": 0, "sample_steps": 0})
        d["ms"] += kms
        d["launches"] += 1
        d["sample_steps"] += samples * nsteps
    dims = P.make_dims(B, n, M, T)
    if not train:
        launches_per_step = P.launch_count(dims, _lib.OP_FORWARD)
    elif world == 1 and not force_collective:  # DataParallelLDBP.step -> ldbp_train_step
        launches_per_step = P.launch_count(dims, _lib.OP_TRAIN_STEP)
    else:  # loss_grad -> all_reduce (NCCL's kernel, not counted) -> adam_kernel
        launches_per_step = P.launch_count(dims, _lib.OP_LOSS_GRAD) + 1
    gpu_launches = launches_per_step * steps

    # e2e: pinned host inputs -> device, step, device -> host read of the result, every step.
    # Double-buffered like a real training loop: step i+1's inputs are copied on a separate copy
    # stream (PCIe) while step i computes; the host still reads every step's result before the
    # next step is launched.
    # Training targets cross PCIe as what a transmitter has: 16-QAM symbol codes (1 byte per symbol)
    # plus per-block power / shift / rotation; the step rebuilds the target waveform on the device
    # (api.ldbp_tx_waveform, the same target as channel.link_blocks) — 1/16 of the bytes of the
    # complex64 target.
    e2e = None
    if want_e2e:
        from paper_2010_14258_b200 import channel

        e2e_steps = max(2, min(steps, 10))
        hx = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for _ in range(2)]
        for i in range(2):
            hx[i].copy_(x)
        dx = [torch.empty_like(x) for _ in range(2)]
        if train:
            codes, pw_b, sh_b, ph_b = channel.link_codes(cfg["idx"], blocks, n)
            qtab = channel.qam16_table(dev)
            hsym = [[torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (codes, pw_b, sh_b, ph_b)]
                    for _ in range(2)]
            for i in range(2):
                for h, t in zip(hsym[i], (codes, pw_b, sh_b, ph_b)):
                    h.copy_(t)
            dsym = [[torch.empty_like(t) for t in (codes, pw_b, sh_b, ph_b)] for _ in range(2)]
            dt = [torch.empty_like(tgt) for _ in range(2)]
            # the device-built target is the one the device-timed steps used
            tchk = P.ldbp_tx_waveform(codes, qtab, pw_b, sps=channel.RHO_D, shift=sh_b, phase=ph_b)
            terr = (torch.linalg.vector_norm(tchk - tgt) / torch.linalg.vector_norm(tgt)).item()
            assert terr < 1e-5, f"device-built targets differ from the bench targets: rel-L2 {terr}"
            del tchk
        else:
            dt = [None, None]
        res = [torch.empty(1 if train else y.numel(), dtype=torch.float64 if train else torch.complex64,
                           pin_memory=True) for _ in range(2)]
        read_ev = [torch.cuda.Event() for _ in range(2)]
        seen = []
        cstream = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]

        def issue_copy(i):
            b = i % 2
            with torch.cuda.stream(cstream):
                cstream.wait_event(freed[b])  # the step that last read buffer b has finished
                dx[b].copy_(hx[b], non_blocking=True)
                if train:
                    for d_, h_ in zip(dsym[b], hsym[b]):
                        d_.copy_(h_, non_blocking=True)
                    # the step's targets from its symbols, on the device, on the copy stream (overlaps
                    # the previous step like the copies do; inside the timed region)
                    P.ldbp_tx_waveform(dsym[b][0], qtab, dsym[b][1], sps=channel.RHO_D, shift=dsym[b][2],
                                       phase=dsym[b][3], out=dt[b], stream=cstream)
                copied[b].record(cstream)

        # the step's kernels on a high-priority stream: the target rebuild on the copy stream then only
        # takes the SM slots the step leaves free (wave tails) instead of sharing them equally
        es = torch.cuda.Stream(device=dev, priority=-1) if os.environ.get("LDBP_BENCH_E2E_PRIO", "1") != "0" else stream
        for b in range(2):
            freed[b].record(stream)
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(es):
            e0.record(es)
            issue_copy(0)
            for i in range(e2e_steps):
                b = i % 2
                es.wait_event(copied[b])
                out = step(dx[b], dt[b])
                freed[b].record(es)
                if i + 1 < e2e_steps:
                    issue_copy(i + 1)  # overlaps this step's compute
                res[b].copy_(out[:1] if train else out.view(-1), non_blocking=True)
                read_ev[b].record(es)
                if i >= 1:  # the host reads step i-1's result while step i runs (no launch bubble)
                    read_ev[1 - b].synchronize()
                    seen.append(float(res[1 - b][0].real))
            read_ev[(e2e_steps - 1) % 2].synchronize()
            seen.append(float(res[(e2e_steps - 1) % 2][0].real))
            e1.record(es)
        torch.cuda.synchronize()
        assert len(seen) == e2e_steps
        e_ms = e0.elapsed_time(e1) / e2e_steps
        if dist.is_initialized():
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        bi = x.numel() * 8 + (sum(t.numel() * t.element_size() for t in hsym[0]) if train else 0)
        bo = 8 if train else y.numel() * 8
        e2e = {"value": samples_global * M / (e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "ms_per_step": round(e_ms, 4),
               "pipeline": "pinned H2D of step i+1 (received samples + transmitted 16-QAM symbol codes) "
                           "and its targets rebuilt on the device (ldbp_tx_waveform) on a copy stream overlap "
                           "step i; result D2H + host read every step"}

    # roofline of the dominant kernel (largest total time)
    sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
    peak_tinst = SMS * FP32_LANES_PER_SM * sm_mhz * 1e6 / 1e12
    peak_max = SMS * FP32_LANES_PER_SM * 1965.0 * 1e6 / 1e12
    dom = max(per_kind.items(), key=lambda kv: kv[1]["ms"]) if per_kind else None
    roof = None
    kernel_shares = {}
    tot_ms = sum(v["ms"] for v in per_kind.values()) or 1.0
    store_all = train and _lib.K_REVERSE in per_kind  # the storing forward of the store-all schedule
    names = {_lib.K_FORWARD: "fwd_store_kernel" if store_all else "fwd_tile_kernel",
             _lib.K_BACKWARD: "bwd_segment_kernel",
             _lib.K_REDUCE: "reduce_partials_kernel+params_kernel" if store_all else "reduce_partials_kernel",
             _lib.K_ADAM: "adam_kernel", _lib.K_REVERSE: "rev_tile_kernel", _lib.K_TINY: "tiny_train_kernel"}
    for k, v in per_kind.items():
        kernel_shares[names[k]] = {"share": round(v["ms"] / tot_ms, 4), "avg_ms": round(v["ms"] / v["launches"], 4),
                                   "launches": v["launches"]}
    if dom:
        kind, v = dom
        ipss = {_lib.K_FORWARD: instr_fwd(kh), _lib.K_TINY: instr_fwd(kh) + instr_bwd(kh)}.get(kind, instr_bwd(kh))
        avg_ms = v["ms"] / v["launches"]
        per_launch_instr = ipss * v["sample_steps"] / v["launches"]
        achieved = per_launch_instr / (avg_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "kernel": names[kind], "achieved": achieved, "peak": peak_tinst,
                "unit": "Tinst/s (FP32 lane-instructions)", "frac": achieved / peak_tinst,
                "frac_at_max_clock": achieved / peak_max, "peak_source": f"148 SM x 128 FP32 lanes x {sm_mhz:.0f} MHz",
                "algorithmic_instr_per_sample_step": ipss, "traffic": traffic_from_profiles(name, names[kind])}
    # whole-step roofline: throughput vs the FP32 bound of the step's algorithmic work
    ips = instr_fwd(kh) + (instr_bwd(kh) if train else 0)
    bound = SMS * FP32_LANES_PER_SM * sm_mhz * 1e6 / ips / 1e9 * world
    step_roof = {"bound_gsample_steps": bound, "frac": value / bound, "instr_per_sample_step": ips}
    return dict(value=value, ms_per_step=ms_per_step, clk=clk, roof=roof, step_roof=step_roof, e2e=e2e,
                gpu_launches=gpu_launches, kernel_shares=kernel_shares, samples_global=samples_global, M=M, T=T,
                B=B, n=n, wall_s=t_wall1 - t_wall0, scaling=scaling, global_blocks=global_blocks(cfg, world, scaling))


def graph_latency(cfg, reps=10, inner=20):
    """Per-step device time with `inner` whole steps (forward, or ldbp_train_step) captured in one
    CUDA graph, replayed back to back (graphs hide the launch cost of C1/C2).  Several
    steps per graph, so that the host's per-replay submission cost (~10 us from Python) is not
    what is measured."""
    import torch

    import paper_2010_14258_b200 as P

    taps, gamma = make_model(cfg)
    x, tgt = make_inputs(cfg, range(cfg["B"]))
    st = P.TrainState.create(taps, gamma)
    ws = P.Workspace()
    train = cfg["mode"] == "train"
    M, T = taps.shape
    buf = torch.empty(1 + M + 2 * M * T, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)

    def step():
        if train:  # the single-process training call (one fused launch when the problem is tiny)
            P.ldbp_train_step(st, x, tgt, buf=buf, ws=ws)
        else:
            P.ldbp_forward(x, st.taps, st.gamma, out=y, ws=ws)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(inner):
            step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * inner) * 1e3  # us


def pipelined_forward(cfg, sets=4, steps=40, warmup=5, graph=True):
    """Serving throughput of the forward (BJ config 2: one forward per batch of received blocks):
    consecutive batches stream through `sets` distinct input/output buffer pairs (4 x 67 MB > the
    126 MB L2, so every batch is read from HBM, no flush needed) with LDBP_STREAM_PIPELINE, so each
    forward's CTAs start while the previous one's last wave drains.  Device time per batch (µs),
    optionally with the `steps` forwards captured in one CUDA graph (PDL edges)."""
    import torch

    import paper_2010_14258_b200 as P

    taps, gamma = make_model(cfg)
    x0, _ = make_inputs(cfg, range(cfg["B"]))
    st = P.TrainState.create(taps, gamma)
    xs = [x0.clone() for _ in range(sets)]
    ys = [torch.empty_like(x0) for _ in range(sets)]

    def run():
        for i in range(steps):
            P.ldbp_forward(xs[i % sets], st.taps, st.gamma, out=ys[i % sets], pipeline=True)

    for _ in range(warmup):
        P.ldbp_forward(xs[0], st.taps, st.gamma, out=ys[0], pipeline=True)
    torch.cuda.synchronize()
    g = None
    if graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        g.replay()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if g is not None:
        g.replay()
    else:
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / steps * 1e3
    # the pipelined outputs are the plain forward's, bit for bit
    ref = P.ldbp_forward(xs[(steps - 1) % sets], st.taps, st.gamma)
    assert torch.equal(ref, ys[(steps - 1) % sets]), "pipelined forward differs from the plain forward"
    return us


def traffic_from_profiles(cfg_name, kernel):
    """dram bytes per launch from a committed `ncu --set full` summary, if one exists."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d[cfg_name][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


# ----------------------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference): the oracle as it stands, on host cores
# ----------------------------------------------------------------------------------------
def _oracle_block(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np

    import ldbp_inputs as li
    from oracle import ldbp as O

    cfg_name, b, taps, gamma, train = args
    cfg = CONFIGS[cfg_name]
    pw = li.dbm_to_w(li.pick_powers_dbm(cfg["idx"], [b], POWERS_DBM))
    x = li.bandlimited_blocks(cfg["idx"], [b], cfg["n"], pw)
    if train:
        t = li.bandlimited_blocks(cfg["idx"], [b], cfg["n"], pw, purpose="target")
        t0 = time.perf_counter()
        O.loss_grad(x, t, taps, gamma, symmetric=True)
    else:
        t0 = time.perf_counter()
        O.forward(x, taps, gamma)
    return time.perf_counter() - t0


def oracle_throughput(cfg_name, target_s, cores, pool=None):
    """Run the oracle over a bounded sample of blocks on `cores` processes; sample-steps/s."""
    import multiprocessing as mp

    import numpy as np

    cfg = CONFIGS[cfg_name]
    taps, gamma = make_model_oracle(cfg)
    taps = taps.astype(np.complex64).astype(np.complex128)
    gamma = gamma.astype(np.float32).astype(np.float64)
    train = cfg["mode"] == "train"
    t1 = _oracle_block((cfg_name, 0, taps, gamma, train))  # calibration (also warms imports)
    nblk = int(max(1, min(cfg["B"], round(target_s * cores / max(t1, 1e-3)))))
    own = pool is None
    pool = pool or mp.get_context("fork").Pool(cores)
    t0 = time.perf_counter()
    pool.map(_oracle_block, [(cfg_name, b, taps, gamma, train) for b in range(nblk)])
    wall = time.perf_counter() - t0
    if own:
        pool.close()
        pool.join()
    M = len(gamma)
    return nblk * cfg["n"] * M / wall / 1e9, nblk, wall


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle timed on this box's host cores (rank 0 only)."""
    import multiprocessing as mp

    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    pool = mp.get_context("fork").Pool(cores)
    per_step_s = 4.0
    vals = []
    for i in range(args.warmup + args.steps):
        v, nblk, wall = oracle_throughput(args.config, per_step_s, cores, pool)
        if i >= args.warmup:
            vals.append((v, nblk, wall))
    pool.close()
    pool.join()
    value = statistics.median(v for v, _, _ in vals)
    nblk = vals[-1][1]
    ms = statistics.median(w for _, _, w in vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling or cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "config": args.config, "B": cfg["B"], "n": cfg["n"],
                   "sample_blocks_per_step": nblk},
        "native_libs_loaded": [l for l in _loaded_libs() if "ldbp" in l],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{nblk} of {cfg['B']} blocks per step (numpy fp64 oracle, process pool)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _loaded_libs():
    try:
        return sorted({ln.split()[-1] for ln in open("/proc/self/maps") if ln.rstrip().endswith(".so")})
    except OSError:
        return []


def _compact(nm, c, rr):
    """Compact per-config summary (the driver keeps only the tail of stdout)."""
    roof = rr["roof"] or {}
    d = {"mode": c["mode"], "value": round(rr["value"], 2), "ms": round(rr["ms_per_step"], 4),
         "kernel": roof.get("kernel"), "kernel_frac": round(roof.get("frac", 0.0), 3),
         "step_frac": round(rr["step_roof"]["frac"], 3), "blocks": rr["global_blocks"], "scaling": rr["scaling"]}
    return d


# ----------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="weak: per-GPU batch fixed (C1-C3 default); strong: global batch fixed (C4, C5 default)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: a functional dry run of the N > 1 path when fewer GPUs than ranks exist "
                         "(ranks share a device; the timings are then not scaling numbers)")
    ap.add_argument("--force-collective", action="store_true",
                    help="N = 1 only: create a one-rank NCCL group and run the data-parallel exchange "
                         "(fp64 all-reduce of the gradient buffer between loss_grad and Adam) every step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (libldbp has no CPU path)")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator lines (ranks, NVLS/P2P transport) for the driver's rank check (NCCL logs to stdout
        # unless NCCL_DEBUG_FILE says otherwise; the JSON line is printed last, after the group is destroyed)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    elif args.force_collective:
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
    import __graft_entry__

    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    import paper_2010_14258_b200  # noqa: F401

    main_cfg = CONFIGS[args.config]
    r = run_config(args.config, main_cfg, args.steps, args.warmup, world, rank, dev, want_e2e=not args.no_e2e,
                   scaling=args.scaling, force_collective=args.force_collective and world == 1)
    extra, detail = {}, {}
    if not args.no_extra:
        for nm in ("C2", "C4", "C5", "C1"):
            if nm == args.config:
                continue
            c = CONFIGS[nm]
            k = 20 if nm in ("C2", "C1") else 10
            rr = run_config(nm, c, k, 3, world, rank, dev, want_e2e=False, want_clocks=False)
            extra[nm] = _compact(nm, c, rr)
            detail[nm] = {"workload": WORKLOAD[nm], "roofline": rr["roof"], "step_roofline": rr["step_roof"],
                          "kernel_shares": rr["kernel_shares"]}
            if nm in ("C1", "C2") and world == 1:  # launch-latency-sensitive: one CUDA graph, replayed
                us = graph_latency(c)
                M = len(make_model(c)[1])
                extra[nm]["graph_us"] = round(us, 2)
                extra[nm]["graph_value"] = round(c["B"] * c["n"] * M / (us * 1e-6) / 1e9, 2)
                if c["mode"] == "fwd":  # serving pipeline of independent batches (LDBP_STREAM_PIPELINE)
                    try:
                        pus = pipelined_forward(c)
                        pv = c["B"] * c["n"] * M / (pus * 1e-6) / 1e9
                        extra[nm]["pipe_us"] = round(pus, 2)
                        extra[nm]["pipe_value"] = round(pv, 2)
                        extra[nm]["pipe_frac"] = round(pv / rr["step_roof"]["bound_gsample_steps"], 3)
                    except Exception as exc:  # an extra: never lose the headline line over it
                        extra[nm]["pipe_error"] = str(exc)[:200]
            torch.cuda.empty_cache()
    cpu = None
    if rank == 0 and not args.no_cpu:
        cores = os.cpu_count() or 1
        v, nblk, wall = oracle_throughput(args.config, 15.0, cores)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{nblk} of {main_cfg['B']} {args.config} blocks, full fwd+bwd (numpy fp64), {wall:.1f} s "
                         f"on a {cores}-process pool"}
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": r["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "dist_backend": args.dist_backend if world > 1 else ("nccl (1 rank, forced exchange)"
                                                                 if args.force_collective else None),
            "extra": extra,
            "config": {"workload": WORKLOAD[args.config], "config": args.config, "blocks_per_gpu": r["B"],
                       "global_blocks": r["global_blocks"], "n": r["n"], "steps_M": r["M"], "taps_T": r["T"],
                       "parallelism": f"dp{world}", "l2": "flushed (256 MiB write) between timed steps",
                       "inputs": "GPU SSFM link 25x80 km, 16-QAM, ASE; pool<=256 blocks shifted/rotated; "
                                 "P in {-2..1} dBm; LS taps"},
            "clocks": r["clk"], "roofline": r["roof"], "step_roofline": r["step_roof"], "cpu_baseline": cpu,
            "e2e": r["e2e"], "gpu_launches": r["gpu_launches"], "kernel_shares": r["kernel_shares"],
        }
        try:
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            with open(os.path.join(ROOT, "gpurun_out", f"bench_detail_n{world}.json"), "w") as fh:
                json.dump({"line": line, "extra_detail": detail}, fh, indent=1)
        except OSError:
            pass
        print(json.dumps({"extra_detail": detail}), file=sys.stderr, flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
