"""Fused tiny training step: device time per step (20 steps per CUDA graph) vs M and cluster cap."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ldbp_inputs as li  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402


def per_step_us(B, n, M, T, inner=20, reps=10):
    x = torch.from_numpy(li.gaussian_blocks(5, range(B), n, 1e-3).astype(np.complex64)).cuda()
    t = torch.from_numpy(li.gaussian_blocks(5, range(B), n, 1e-3, purpose="target").astype(np.complex64)).cuda()
    st = P.TrainState.create(li.random_sym_taps(5, M, T, 0.1), li.random_gamma(5, M))
    buf = torch.empty(1 + M + 2 * M * T, dtype=torch.float64, device="cuda")
    ws = P.Workspace()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            P.ldbp_train_step(st, x, t, buf=buf, ws=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(inner):
            P.ldbp_train_step(st, x, t, buf=buf, ws=ws)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * inner) * 1e3


for (B, n, T) in ((4, 1024, 3), (1, 4096, 3), (8, 1024, 3)):
    for M in (1, 2, 4, 8, 16):
        row = []
        for env in ({"LDBP_TINY": "0"}, {"LDBP_TINY_MAX_CLUSTER": str(B)}, {"LDBP_TINY_MAX_CLUSTER": str(min(8, 2 * B))},
                    {"LDBP_TINY_MAX_CLUSTER": "16"}):
            for k in ("LDBP_TINY", "LDBP_TINY_MAX_CLUSTER"):
                os.environ.pop(k, None)
            os.environ.update(env)
            row.append("%s=%.2f" % (",".join(f"{k[5:]}:{v}" for k, v in env.items()), per_step_us(B, n, M, T)))
        print(f"B={B} n={n} T={T} M={M}: " + "  ".join(row), flush=True)
