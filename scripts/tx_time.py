"""Device time of ldbp_tx_waveform at the C3 batch (512 blocks x 2^14) and of the C3 training step
with and without a concurrent tx_waveform on a second stream (the e2e pipeline's overlap cost)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_14258_b200 as P  # noqa: E402
from paper_2010_14258_b200 import channel  # noqa: E402

cfg = bench.CONFIGS["C3"]
B, n = cfg["B"], cfg["n"]
codes, pw, sh, ph = channel.link_codes(cfg["idx"], range(B), n)
q = channel.qam16_table()
out = torch.empty((B, n), dtype=torch.complex64, device="cuda")


def tx(stream=None):
    P.ldbp_tx_waveform(codes, q, pw, sps=channel.RHO_D, shift=sh, phase=ph, out=out, stream=stream)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print(f"tx_waveform alone: {timed(tx):.4f} ms")
taps, gamma = bench.make_model(cfg)
x, tgt = bench.make_inputs(cfg, range(B))
st = P.TrainState.create(taps, gamma)
buf = torch.empty(1 + st.taps.shape[0] * (1 + 2 * st.taps.shape[1]), dtype=torch.float64, device="cuda")
step = lambda: P.ldbp_train_step(st, x, tgt, buf=buf)  # noqa: E731
print(f"train step alone: {timed(step):.4f} ms")
s2 = torch.cuda.Stream()


def both():
    s2.wait_stream(torch.cuda.current_stream())
    tx(stream=s2)
    step()
    torch.cuda.current_stream().wait_stream(s2)


print(f"train step + concurrent tx_waveform: {timed(both):.4f} ms")
