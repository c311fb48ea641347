"""Kernel-time sweep for tuning: python scripts/quick_bench.py C2 [C4 ...] (env vars select plans)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402
from paper_2010_14258_b200 import _lib  # noqa: E402

names = sys.argv[1:] or ["C2", "C4", "C3", "C5"]
for name in names:
    cfg = bench.CONFIGS[name]
    taps, gamma = bench.make_model(cfg)
    x, tgt = bench.make_inputs(cfg, range(cfg["B"]))
    st = P.TrainState.create(taps, gamma)
    M, T = taps.shape
    kh = (T - 1) // 2
    train = cfg["mode"] == "train"
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ws = P.Workspace()

    def step():
        if train:
            return P.ldbp_loss_grad(x, tgt, st.taps, st.gamma, ws=ws)
        return P.ldbp_forward(x, st.taps, st.gamma, ws=ws)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    reps = 10
    # wall time of the whole step (CUDA events on the calling stream; valid with internal overlap)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i in range(reps):
        flush.fill_(i)
        evs[i][0].record()
        step()
        evs[i][1].record()
    torch.cuda.synchronize()
    wall = sum(a.elapsed_time(b) for a, b in evs) / reps
    per = {}
    tot = 0.0
    with P.api.trace() as tr:
        for i in range(reps):
            flush.fill_(i)
            step()
        torch.cuda.synchronize()
    for kind, steps, samples, ms in tr.records:
        d = per.setdefault(kind, [0.0, 0, 0])
        d[0] += ms
        d[1] += 1
        d[2] += samples * steps
        tot += ms
    ms_step = tot / reps
    ss = cfg["B"] * cfg["n"] * M
    ips = bench.instr_fwd(kh) + (bench.instr_bwd(kh) if train else 0)
    peak = 148 * 128 * 1.965e9
    print(f"{name}: wall {wall:.3f} ms/step  {ss / wall / 1e6:.1f} Gss/s  step-frac@1965 {ss * ips / (wall * 1e-3) / peak:.3f}"
          f"  (sum of traced kernel times {ms_step:.3f} ms)")
    for kind, (ms, nl, sst) in sorted(per.items()):
        ipss = bench.instr_fwd(kh) if kind == _lib.K_FORWARD else bench.instr_bwd(kh) if kind in (_lib.K_BACKWARD, _lib.K_REVERSE) else 0
        frac = (ipss * sst / (ms * 1e-3) / peak) if ipss else 0
        print(f"   kind {kind}: {ms / reps:.3f} ms/step over {nl // reps} launches, frac {frac:.3f}")
    del x, tgt, ws
    torch.cuda.empty_cache()
