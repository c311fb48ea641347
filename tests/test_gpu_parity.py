"""GPU-vs-oracle parity of the CUDA path through the C ABI (SURVEY.md §8(c) "the gate").

Tolerances (BASELINE.json north_star): outputs rel-L2 <= 1e-5 per block; gradients rel-L2 <=
1e-4 per step for taps and for gamma' separately; loss <= 1e-5; effective SNR +-0.01 dB.
The oracle runs on the same fp32-rounded inputs in complex128.
"""
import numpy as np
import pytest
import torch

import ldbp_inputs as li
from oracle import channel, ldbp as O, physics, receiver, steps

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-5
GRAD_TOL = 1e-4


@pytest.fixture(scope="module")
def P():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2010_14258_b200 as P

    return P


def dev(a, dtype=np.complex64):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).astype(dtype))).cuda()


def r32(a):
    """What the GPU sees, promoted for the oracle."""
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return a.astype(np.complex64).astype(np.complex128)
    return a.astype(np.float32).astype(np.float64)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def model(cfg, M, T, sym, scale=0.1, ls=False, sub=0):
    if ls:
        _, g = steps.dbp_plan(M, 80.0, 1, 0.2, 1.3)
        xi = [steps.xi_of(80.0, physics.ps2_per_km(-21.7), 21.4e9)] * M
        taps = np.stack([steps.ls_taps(x, T, cap=1.0) for x in xi])
        return taps, g
    taps = li.random_sym_taps(cfg, M, T, scale) if sym else li.random_general_taps(cfg, M, T, scale, sub=sub)
    gamma = li.random_gamma(cfg, M, sub=sub)
    return taps, gamma


FWD_CASES = [
    # (B, n, M, T, sym, power_w)
    (4, 1024, 4, 3, True, 1e-3),     # C1 shape
    (3, 1000, 6, 5, True, 1e-3),     # ragged n (not a multiple of the per-thread chunk)
    (2, 777, 3, 9, False, 1e-3),     # general (non-symmetric) taps, odd n
    (1, 5, 2, 5, True, 1e-3),        # n == T
    (2, 16, 10, 7, True, 1e-3),      # halo H = 30 > n: multiple wraps
    (2, 64, 1, 1, True, 1e-3),       # T = 1 (pointwise), M = 1
    (5, 4099, 12, 15, True, 1e-3),   # Kh = 7, several tiles, ragged tail
    (3, 3000, 7, 13, False, 2e-3),   # Kh = 6 general
    (1, 9000, 5, 11, True, 1e-3),
]


@pytest.mark.parametrize("B,n,M,T,sym,pw", FWD_CASES)
def test_forward_parity(P, B, n, M, T, sym, pw):
    x = li.gaussian_blocks(11, range(B), n, pw)
    taps, gamma = model(11, M, T, sym)
    y = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32), symmetric=sym).cpu().numpy()
    ref = O.forward(r32(x), r32(taps), r32(gamma))
    for b in range(B):
        assert rel(y[b], ref[b]) <= OUT_TOL, (b, rel(y[b], ref[b]))


def test_forward_precise_flag(P):
    B, n, M, T = 3, 2500, 8, 5
    x = li.gaussian_blocks(12, range(B), n, 2e-3)
    taps, gamma = model(12, M, T, True)
    ref = O.forward(r32(x), r32(taps), r32(gamma))
    yp = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32), precise=True).cpu().numpy()
    yf = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32)).cpu().numpy()
    assert rel(yp, ref) <= 2e-6 and rel(yf, ref) <= OUT_TOL


@pytest.mark.parametrize("cmax", [None, "3"])
def test_forward_stream_pipeline(P, monkeypatch, cmax):
    """LDBP_STREAM_PIPELINE: back-to-back forwards of independent batches over a rotation of 3
    buffer pairs (programmatic dependent launches, no wait on the previous grid) give the oracle's
    outputs and the plain forward's bits; a multi-launch forward (cmax = 3) ignores the flag."""
    if cmax:
        monkeypatch.setenv("LDBP_FWD_MAX_STEPS", cmax)
    B, n, M, T = 5, 3000, 7, 5
    taps, gamma = model(14, M, T, True)
    xs = [li.gaussian_blocks(14, range(k * B, (k + 1) * B), n, 2e-3) for k in range(3)]
    dx = [dev(x) for x in xs]
    ys = [torch.empty_like(d) for d in dx]
    tt, gg = dev(taps), dev(gamma, np.float32)
    for it in range(4):
        for k in range(3):
            P.ldbp_forward(dx[k], tt, gg, out=ys[k], pipeline=True)
    for k in range(3):
        plain = P.ldbp_forward(dx[k], tt, gg)
        assert torch.equal(plain, ys[k]), k
        ref = O.forward(r32(xs[k]), r32(taps), r32(gamma))
        y = ys[k].cpu().numpy()
        for b in range(B):
            assert rel(y[b], ref[b]) <= OUT_TOL, (k, b)


def test_forward_chained_launches(P, monkeypatch):
    """Force several launches per forward (checkpoint-style chaining through the workspace)."""
    B, n, M, T = 3, 1500, 10, 5
    x = li.gaussian_blocks(13, range(B), n, 1e-3)
    taps, gamma = model(13, M, T, True)
    ref = O.forward(r32(x), r32(taps), r32(gamma))
    for cmax in ("3", "4", "10"):
        monkeypatch.setenv("LDBP_FWD_MAX_STEPS", cmax)
        y = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32)).cpu().numpy()
        assert rel(y, ref) <= OUT_TOL, cmax


def test_delay_taps_closed_form(P):
    """P9: h^(i) = e^{j th_i} delta_{j_i} (general path) gives
    y_t = x_{t-S} exp(j(sum th + sum gamma' |x_{t-S}|^2)) — exercises halos and the wrap."""
    B, n, T = 3, 4099, 7
    shifts, th = [3, -2, 3, 1, -3], [0.3, -1.1, 2.0, 0.2, 0.9]
    M = len(shifts)
    taps = np.zeros((M, T), complex)
    for i, (j, t) in enumerate(zip(shifts, th)):
        taps[i, j + 3] = np.exp(1j * t)
    gamma = np.array([-20.0, 15.0, -30.0, 10.0, -5.0])
    x = li.gaussian_blocks(14, range(B), n, 2e-3)
    y = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32), symmetric=False).cpu().numpy()
    xs = np.roll(r32(x), sum(shifts), axis=-1)
    ref = xs * np.exp(1j * (np.sum(th) + r32(gamma).sum() * np.abs(xs) ** 2))
    assert rel(y, ref) <= 1e-6


def test_equivariance_c2_size(P):
    """P10 at the C2 size: f(shift_k(e^{j phi} x)) = shift_k(e^{j phi} f(x))."""
    B, n, M, T = 256, 16384, 25, 5
    x = li.bandlimited_blocks_torch(1, B, n, 1e-3)
    taps, gamma = model(0, M, T, True, ls=True)
    ht, gt = dev(taps), dev(gamma, np.float32)
    y = P.ldbp_forward(x, ht, gt)
    k, phi = 4321, 0.7
    rot = torch.tensor(np.exp(1j * phi), dtype=torch.complex64, device="cuda")
    y2 = P.ldbp_forward(torch.roll(x * rot, k, dims=1).contiguous(), ht, gt)
    ref = torch.roll(y * rot, k, dims=1)
    err = (torch.linalg.vector_norm(y2 - ref, dim=1) / torch.linalg.vector_norm(ref, dim=1)).max().item()
    assert err <= 1e-6


BWD_CASES = [
    # (B, n, M, T, sym, max_steps_env)
    (4, 1024, 4, 3, True, None),   # C1
    (3, 1000, 6, 5, True, "2"),    # 3 segments
    (2, 700, 5, 7, False, "3"),    # general, 2 uneven segments
    (2, 40, 7, 9, True, "3"),      # H > n
    (2, 300, 3, 1, True, None),    # T = 1
    (3, 2100, 9, 15, True, "4"),
]


# the two row-a7 schedules: 0 = checkpoint + recompute segments, 1 = store-all + fused reverse;
# "1r4" = store-all with the shared-memory-adjoint reverse kernel (ldbp_reverse4.cuh), "1rt" = with
# the register-resident one (rev_tile_kernel)
MODES = ["0", "1", "1r4", "1rt"]


def set_mode(monkeypatch, mode, cmax):
    if mode.startswith("1r"):
        monkeypatch.setenv("LDBP_REV4", "1" if mode == "1r4" else "0")
        monkeypatch.setenv("LDBP_STORE_ALL_MIN_SAMPLES", "0")
        mode = "1"
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_TINY", "0")  # the schedule under test, not the fused C1 kernel
    if cmax:
        monkeypatch.setenv("LDBP_BWD_MAX_STEPS", cmax)
        monkeypatch.setenv("LDBP_REV_MAX_STEPS", cmax)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("B,n,M,T,sym,cmax", BWD_CASES)
def test_backward_parity(P, monkeypatch, B, n, M, T, sym, cmax, mode):
    set_mode(monkeypatch, mode, cmax)
    x = li.gaussian_blocks(21, range(B), n, 1e-3)
    gy = li.gaussian_blocks(21, range(B), n, 1.0, purpose="grad")
    taps, gamma = model(21, M, T, sym)
    dt, dg, gx = P.ldbp_backward(dev(x), dev(gy), dev(taps), dev(gamma, np.float32), symmetric=sym)
    rdt, rdg, rgx = O.backward(r32(x), r32(gy), r32(taps), r32(gamma))
    if sym:
        rdt = O.sym_fold(rdt)
    dt, dg, gx = dt.cpu().numpy(), dg.cpu().numpy(), gx.cpu().numpy()
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= GRAD_TOL, (i, rel(dt[i], rdt[i]))
        assert abs(dg[i] - rdg[i]) <= GRAD_TOL * abs(rdg[i]) + 1e-12 * np.abs(rdg).max(), (i, dg[i], rdg[i])
    for b in range(B):
        assert rel(gx[b], rgx[b]) <= OUT_TOL * 10, (b, rel(gx[b], rgx[b]))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("sym,masked,cmax", [(True, False, None), (True, True, "2"), (False, True, None)])
def test_loss_grad_parity(P, monkeypatch, sym, masked, cmax, mode):
    set_mode(monkeypatch, mode, cmax)
    B, n, M, T = 4, 1536, 6, 9
    x = li.gaussian_blocks(31, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(31, range(B), n, 1e-3, purpose="target")
    taps, gamma = model(31, M, T, sym)
    mask = None
    if masked:
        mask = np.ones((M, T), np.uint8)
        mask[1, [0, 8]] = 0
        mask[4, [0, 1, 7, 8]] = 0
    buf = P.ldbp_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32), symmetric=sym,
                           mask=None if mask is None else torch.from_numpy(mask).cuda()).cpu().numpy()
    ref = O.loss_grad(r32(x), r32(tgt), r32(taps), r32(gamma), mask=mask, symmetric=sym)
    assert abs(buf[0] - ref[0]) <= OUT_TOL * ref[0]
    for i in range(M):  # dgamma'_i per step (a scalar each)
        assert abs(buf[1 + i] - ref[1 + i]) <= GRAD_TOL * abs(ref[1 + i]), (i, buf[1 + i], ref[1 + i])
    dt, rdt = buf[1 + M:].reshape(M, T, 2), ref[1 + M:].reshape(M, T, 2)
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= GRAD_TOL, i
    if masked:
        assert np.all(dt[mask == 0] == 0)


@pytest.mark.parametrize("mode", MODES)
def test_gradient_gauge_identities_gpu(P, monkeypatch, mode):
    """P6/P7 on the GPU gradients (Remark 4): exact in exact arithmetic, <= 1e-4 relative here."""
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_TINY", "0")
    B, n, M, T = 8, 4096, 10, 5
    x = li.gaussian_blocks(41, range(B), n, 2e-3)
    tgt = li.gaussian_blocks(41, range(B), n, 2e-3, purpose="target")
    taps, gamma = model(41, M, T, False)
    buf = P.ldbp_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32), symmetric=False).cpu().numpy()
    dg = buf[1:1 + M]
    dt = buf[1 + M:].reshape(M, T, 2)
    dt = dt[..., 0] + 1j * dt[..., 1]
    h = r32(taps)
    g32 = r32(gamma)
    ip = [np.sum(np.conj(dt[i]) * h[i]) for i in range(M)]
    mag = max(max(abs(v) for v in ip), np.max(np.abs(2 * g32 * dg)))
    for i in range(M - 1):
        assert abs(ip[i + 1].real - ip[i].real + 2 * g32[i] * dg[i]) <= 1e-4 * mag
        assert abs(ip[i].imag - ip[i + 1].imag) <= 1e-4 * mag


def test_adam_parity_same_gradient(P):
    """G13: GPU Adam vs oracle Adam fed the same gradient buffer (<= 1e-12 rel in fp64 master)."""
    M, T = 5, 9
    taps, gamma = model(51, M, T, True)
    mask = np.ones((M, T), np.uint8)
    mask[2, [0, 8]] = 0
    gl = np.array([1, 1, 0, 1, 1], np.uint8)
    st = P.TrainState.create(taps, gamma, mask=mask, gamma_learnable=gl)
    theta = O.pack_params(taps, gamma)
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    rng = np.random.default_rng(5)
    for t in range(1, 4):
        buf = rng.standard_normal(1 + M + 2 * M * T) * 10.0 ** rng.uniform(-6, 2, 1 + M + 2 * M * T)
        P.ldbp_adam_update(st, torch.from_numpy(buf).cuda(), 12345.0)
        theta, m, v = O.adam_update(buf, 12345.0, theta, m, v, t, M, T, tap_mask=mask, gamma_learnable=gl)
        assert rel(st.master.cpu().numpy(), theta) <= 1e-12
        assert rel(st.m.cpu().numpy(), m) <= 1e-12 and rel(st.v.cpu().numpy(), v) <= 1e-12
    w = st.taps.cpu().numpy()
    th_t, th_g = O.unpack_params(theta, M, T)
    np.testing.assert_array_equal(w, th_t.astype(np.complex64))
    np.testing.assert_array_equal(st.gamma.cpu().numpy(), th_g.astype(np.float32))


def test_train_step_is_loss_grad_plus_adam(P):
    B, n, M, T = 3, 2048, 5, 5
    x = dev(li.gaussian_blocks(61, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(61, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(61, M, T, True)
    s1 = P.TrainState.create(taps, gamma)
    s2 = P.TrainState.create(taps, gamma)
    for _ in range(3):
        b1 = P.ldbp_train_step(s1, x, tgt)
        b2 = P.ldbp_loss_grad(x, tgt, s2.taps, s2.gamma)
        P.ldbp_adam_update(s2, b2, B * n)
        assert torch.equal(b1, b2)
    # same gradient; Adam in the fused tiny kernel (C1-sized problems) or adam_kernel: the same
    # adam_elem arithmetic, compiled into two kernels (fp64 contraction may differ by an ulp)
    assert rel(s1.master.cpu().numpy(), s2.master.cpu().numpy()) <= 1e-14
    assert rel(s1.taps.cpu().numpy(), s2.taps.cpu().numpy()) <= 1e-7


@pytest.mark.parametrize("mode", MODES)
def test_determinism_and_shard_sum(P, monkeypatch, mode):
    """Fixed-order reductions: bitwise repeatable; the data-parallel sum of per-shard buffers
    equals the full-batch buffer (gradient is linear in the blocks; §8(e))."""
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_TINY", "0")
    B, n, M, T = 8, 3000, 6, 5
    x = li.gaussian_blocks(71, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(71, range(B), n, 1e-3, purpose="target")
    taps, gamma = model(71, M, T, True)
    ht, gt = dev(taps), dev(gamma, np.float32)
    full = P.ldbp_loss_grad(dev(x), dev(tgt), ht, gt)
    again = P.ldbp_loss_grad(dev(x), dev(tgt), ht, gt)
    assert torch.equal(full, again)
    parts = sum(P.ldbp_loss_grad(dev(x[s:s + 2]), dev(tgt[s:s + 2]), ht, gt).cpu().numpy() for s in range(0, B, 2))
    assert rel(parts, full.cpu().numpy()) <= 1e-6


def _inband_unit_taps(T, band=0.275):
    """LS inverse-CD taps for one 80 km step fitted in band (10% RRC at 2 sps occupies |f| <= 0.275
    f_s) and normalised to unit mean in-band gain — an init-quality stand-in so that the 1-StPS
    receiver is a working equaliser in this test (the taps are an input; parity is unaffected)."""
    xi = steps.xi_of(80.0, physics.ps2_per_km(-21.7), 21.4e9)
    h = steps.ls_taps(xi, T, band=band, oob_weight=0.3)
    w = np.linspace(-2 * np.pi * band, 2 * np.pi * band, 2001)
    k = np.arange(T) - (T - 1) // 2
    return h / np.sqrt(np.mean(np.abs(np.exp(-1j * np.outer(w, k)) @ h) ** 2))


def test_snr_parity_on_simulated_link(P):
    """Effective SNR after LDBP (oracle receiver on both outputs) agrees to 0.01 dB, on seeded
    SSFM + EDFA blocks of the C2 link (25 x 80 km, 1 StPS, n = 2^14 samples = 8192 symbols per
    block) at all 11 launch powers -4..+6 dBm, for the C2 filter length (T = 5)
    and a working in-band equaliser (T = 15), with and without the nonlinear steps."""
    nsym, spans, M, nblk = 8192, 25, 25, 2
    link = dict(span_km=80.0, alpha_db=0.2, beta2=physics.ps2_per_km(-21.7), gamma=1.3, baud_hz=10.7e9,
                rho_a=4, rho_d=2, nf_db=5.0, nu_hz=1.946e14)
    _, gam = steps.dbp_plan(spans, 80.0, 1, 0.2, 1.3)
    snr = {}
    for pdbm in [float(p) for p in range(-4, 7)]:
        pw = float(physics.dbm_to_w(pdbm))
        rs, ss = [], []
        for b in range(nblk):
            s = li.qam16(li.rng(2, b, "symbols", sub=int(pdbm + 10)), nsym)
            ase = [li.cn(li.rng(2, b, "ase", sub=100 * int(pdbm + 10) + k), nsym * 4) for k in range(spans)]
            r, _ = channel.simulate_link(s, pw, num_spans=spans, steps_per_span=8, ase_draws=ase, **link)
            rs.append(r)
            ss.append(s)
        rs = np.array(rs)
        for T in (5, 15):
            taps = np.stack([_inband_unit_taps(T)] * M)
            for nl in (True, False):
                g = gam if nl else 0 * gam
                y = P.ldbp_forward(dev(rs), dev(taps), dev(g, np.float32)).cpu().numpy()
                yo = O.forward(r32(rs), r32(taps), r32(g))
                snr_gpu = receiver.evaluate(y.astype(np.complex128), ss, [pw] * nblk)
                snr_ref = receiver.evaluate(yo, ss, [pw] * nblk)
                assert abs(snr_gpu[0] - snr_ref[0]) <= 0.01, (pdbm, T, nl, snr_gpu, snr_ref)
                assert abs(snr_gpu[1] - snr_ref[1]) <= 0.01, (pdbm, T, nl, snr_gpu, snr_ref)
                snr[(pdbm, T, nl)] = snr_gpu[0]
    # the T = 15 receiver equalises, and its nonlinear steps help at high power (DBP works)
    assert snr[(-4.0, 15, True)] > 12.0
    assert snr[(2.0, 15, True)] > snr[(2.0, 15, False)] + 3.0
    assert snr[(6.0, 15, True)] > snr[(6.0, 15, False)] + 3.0


@pytest.mark.parametrize("mode", MODES)
def test_backward_unnormalised_path(P, monkeypatch, mode):
    """Taps whose centre tap is ~0 make the h0-normalised kernels fall back to the plain folded
    FIR (launch-wide, decided on the device); gradients must still match the oracle."""
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_TINY", "0")
    B, n, M, T = 2, 900, 4, 5
    x = li.gaussian_blocks(81, range(B), n, 1e-3)
    gy = li.gaussian_blocks(81, range(B), n, 1.0, purpose="grad")
    taps, gamma = model(81, M, T, True)
    taps[2, 2] = 1e-6  # h0 of step 2 ~ 0 -> not normalisable
    y = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32)).cpu().numpy()
    assert rel(y, O.forward(r32(x), r32(taps), r32(gamma))) <= OUT_TOL
    dt, dg, gx = P.ldbp_backward(dev(x), dev(gy), dev(taps), dev(gamma, np.float32))
    rdt, rdg, rgx = O.backward(r32(x), r32(gy), r32(taps), r32(gamma))
    rdt = O.sym_fold(rdt)
    dt, dg = dt.cpu().numpy(), dg.cpu().numpy()
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= GRAD_TOL, i
    assert rel(dg, rdg) <= GRAD_TOL
    assert rel(gx.cpu().numpy(), rgx) <= 1e-4


@pytest.mark.parametrize("mode", MODES)
def test_precise_backward(P, monkeypatch, mode):
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_TINY", "0")
    B, n, M, T = 2, 1200, 5, 7
    x = li.gaussian_blocks(82, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(82, range(B), n, 1e-3, purpose="target")
    taps, gamma = model(82, M, T, True)
    buf = P.ldbp_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32), precise=True).cpu().numpy()
    ref = O.loss_grad(r32(x), r32(tgt), r32(taps), r32(gamma), symmetric=True)
    assert abs(buf[0] - ref[0]) <= 1e-6 * ref[0]
    assert rel(buf[1:], ref[1:]) <= 2e-5


def test_train_step_cuda_graph_capture(P):
    """The ABI promises no host sync inside calls: a whole training step (loss_grad + Adam) is
    captured in a CUDA graph and replayed; results equal eager execution."""
    B, n, M, T = 4, 2048, 6, 9
    x = dev(li.gaussian_blocks(83, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(83, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(83, M, T, True)
    eager = P.TrainState.create(taps, gamma)
    graphed = P.TrainState.create(taps, gamma)
    ws = P.Workspace()
    buf = torch.empty(1 + M + 2 * M * T, dtype=torch.float64, device="cuda")
    # warm up on a side stream (allocates the workspace), then capture one step
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        P.ldbp_loss_grad(x, tgt, graphed.taps, graphed.gamma, buf=buf, ws=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        P.ldbp_loss_grad(x, tgt, graphed.taps, graphed.gamma, buf=buf, ws=ws)
        P.ldbp_adam_update(graphed, buf, B * n)
    graphed.t = 0  # capture advanced the host-side counter; the captured launch uses t = 1
    for it in range(3):
        b_e = P.ldbp_loss_grad(x, tgt, eager.taps, eager.gamma)
        P.ldbp_adam_update(eager, b_e, B * n)
        g.replay()
        torch.cuda.synchronize()
        if it == 0:
            assert torch.equal(b_e, buf)
            assert torch.equal(eager.master, graphed.master)


@pytest.mark.parametrize("masked", [False, True])
def test_store_all_param_table_in_global_memory(P, monkeypatch, masked):
    """Models longer than kParamsSmemSteps (3072) build the store-all parameter table with the
    prefix-product chain in global memory instead of shared memory; forced here for a short model
    (LDBP_PARAMS_SMEM_STEPS=0): identical arithmetic, so results equal the default path exactly.
    (Long random models are not used for parity: their fp32 rounding differences grow
    exponentially with M — measured 1.4e-5 at M = 100, O(1) at M = 1000 — for any schedule.)"""
    monkeypatch.setenv("LDBP_BWD_MODE", "1")
    B, n, M, T = 3, 4096, 12, 9
    x = dev(li.gaussian_blocks(97, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(97, range(B), n, 1e-3, purpose="target"))
    taps, gamma, mask = pruned_model(97, M, T, [4, 3, 4, 2, 4, 4, 1, 4, 3, 4, 4, 2])
    mk = torch.from_numpy(mask).cuda() if masked else None
    ref_buf = P.ldbp_loss_grad(x, tgt, dev(taps), dev(gamma, np.float32), mask=mk)
    monkeypatch.setenv("LDBP_PARAMS_SMEM_STEPS", "0")
    buf = P.ldbp_loss_grad(x, tgt, dev(taps), dev(gamma, np.float32), mask=mk)
    assert torch.equal(buf, ref_buf)
    ref = O.loss_grad(r32(x.cpu().numpy()), r32(tgt.cpu().numpy()), r32(taps), r32(gamma),
                      mask=mask if masked else None, symmetric=True)
    b = buf.cpu().numpy()
    assert abs(b[0] - ref[0]) <= OUT_TOL * ref[0]
    assert rel(b[1:], ref[1:]) <= GRAD_TOL


@pytest.mark.parametrize("mode", MODES)
def test_launch_count_matches_traced_launches(P, monkeypatch, mode):
    """ldbp_launch_count (the bench's gpu_launches claim) equals the launches the library actually
    makes for one loss_grad + Adam step, in both schedules (store-all adds params_kernel)."""
    set_mode(monkeypatch, mode, None)
    B, n, M, T = 64, 16384, 6, 9  # B*n = 2^20: store-all eligible
    x = dev(li.gaussian_blocks(91, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(91, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(91, M, T, True)
    st = P.TrainState.create(taps, gamma)
    buf = P.ldbp_loss_grad(x, tgt, st.taps, st.gamma)  # warm-up (workspace)
    torch.cuda.synchronize()
    with P.api.trace() as tr:
        buf = P.ldbp_loss_grad(x, tgt, st.taps, st.gamma)
        P.ldbp_adam_update(st, buf, B * n)
        torch.cuda.synchronize()
    d = P.make_dims(B, n, M, T)
    assert len(tr.records) == P.launch_count(d, P._lib.OP_TRAIN_STEP)


# ---- §8(f) NEXT-3: per-step variable filter lengths (pruned outer taps are not computed) ----
def pruned_model(seed, M, T, kh_steps):
    """Symmetric taps whose step i keeps only |j| <= kh_steps[i] (progressive pruning
    removes the outermost pair; Example 2's models alternate lengths)."""
    taps, gamma = model(seed, M, T, True)
    kh = (T - 1) // 2
    mask = np.ones((M, T), np.uint8)
    for i, k in enumerate(kh_steps):
        for j in range(k + 1, kh + 1):
            mask[i, kh + j] = mask[i, kh - j] = 0
    return taps * mask, gamma, mask


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("B,n,M,T,kh_steps", [
    (3, 4096, 8, 9, [4, 3, 2, 1, 0, 4, 2, 3]),   # every active length incl. below KH-2 (fallback variant)
    (2, 3000, 6, 5, [2, 1, 2, 1, 2, 1]),         # alternating 5/3 taps (Example 2 pattern)
    (2, 2048, 5, 15, [7, 6, 5, 3, 7]),
])
def test_variable_tap_lengths(P, monkeypatch, mode, B, n, M, T, kh_steps):
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_TINY", "0")
    monkeypatch.setenv("LDBP_STORE_ALL_MIN_SAMPLES", "0")
    taps, gamma, mask = pruned_model(91, M, T, kh_steps)
    x = li.gaussian_blocks(91, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(91, range(B), n, 1e-3, purpose="target")
    # forward: zero outer taps (no mask argument) -> skipped per step, result as the oracle's
    y = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32)).cpu().numpy()
    yr = O.forward(r32(x), r32(taps), r32(gamma))
    for b in range(B):
        assert rel(y[b], yr[b]) <= OUT_TOL, b
    # training gradient with the pruning mask: masked taps get exactly 0, the rest match
    buf = P.ldbp_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32),
                           mask=torch.from_numpy(mask).cuda()).cpu().numpy()
    ref = O.loss_grad(r32(x), r32(tgt), r32(taps), r32(gamma), mask=mask, symmetric=True)
    assert abs(buf[0] - ref[0]) <= OUT_TOL * ref[0]
    assert rel(buf[1:1 + M], ref[1:1 + M]) <= GRAD_TOL
    dt, rdt = buf[1 + M:].reshape(M, T, 2), ref[1 + M:].reshape(M, T, 2)
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= GRAD_TOL, i
    assert np.all(dt[mask == 0] == 0)


@pytest.mark.parametrize("mode", MODES)
def test_sharding_bit_identity(P, monkeypatch, mode):
    """§8(e): forward outputs are bit-identical for any partition of the blocks across ranks (each
    output sample's arithmetic does not depend on the tiling), and the unreduced gradient buffers
    of the shards sum to the full buffer up to the grouping of the per-CTA fp32 partial sums (the
    tiles differ between shardings; every grouping is a valid fp32 sum, ~1e-9 apart)."""
    monkeypatch.setenv("LDBP_BWD_MODE", mode)
    monkeypatch.setenv("LDBP_TINY", "0")
    monkeypatch.setenv("LDBP_STORE_ALL_MIN_SAMPLES", "0")
    B, n, M, T = 8, 6000, 10, 9
    x = dev(li.gaussian_blocks(95, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(95, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(95, M, T, True)
    ht, gt = dev(taps), dev(gamma, np.float32)
    y = P.ldbp_forward(x, ht, gt)
    for parts in ((4, 4), (2, 2, 2, 2), (1, 7), (3, 5)):
        o = 0
        for p in parts:
            ys = P.ldbp_forward(x[o:o + p].contiguous(), ht, gt)
            assert torch.equal(ys, y[o:o + p]), (parts, o)
            o += p
    full = P.ldbp_loss_grad(x, tgt, ht, gt).cpu().numpy()
    sh = sum(P.ldbp_loss_grad(x[o:o + 4].contiguous(), tgt[o:o + 4].contiguous(), ht, gt).cpu().numpy()
             for o in (0, 4))
    assert rel(sh, full) <= 1e-7


def test_check_finite_reports_first_step(P, monkeypatch):
    """LDBP_CHECK_FINITE (§8(b)): finite runs pass and give the unchecked result; a
    model whose step 3 overflows fp32 (taps 1e25 there) fails with LDBP_ENONFINITE naming step 3,
    for the forward and for the training gradient."""
    from paper_2010_14258_b200 import LdbpError

    B, n, M, T = 2, 2048, 6, 5
    x = dev(li.gaussian_blocks(97, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(97, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(97, M, T, True)
    ht, gt = dev(taps), dev(gamma, np.float32)
    assert torch.equal(P.ldbp_forward(x, ht, gt, check_finite=True), P.ldbp_forward(x, ht, gt))
    monkeypatch.setenv("LDBP_BWD_MODE", "1")  # checked training calls run the store-all schedule
    monkeypatch.setenv("LDBP_TINY", "0")  # (the unchecked call too, so that both are the same schedule)
    assert torch.equal(P.ldbp_loss_grad(x, tgt, ht, gt, check_finite=True), P.ldbp_loss_grad(x, tgt, ht, gt))
    bad = taps.copy()
    bad[2] *= 1e25  # |a| ~ 1e22 after step 3: |a|^2 overflows -> NaN phase
    hb = dev(bad)
    with pytest.raises(LdbpError) as e:
        P.ldbp_forward(x, hb, gt, check_finite=True)
    assert e.value.status == -6 and "step 3" in str(e.value)
    with pytest.raises(LdbpError) as e:
        P.ldbp_loss_grad(x, tgt, hb, gt, check_finite=True)
    assert e.value.status == -6 and "step 3" in str(e.value)


@pytest.mark.parametrize("env", [{"LDBP_BWD_MODE": "1"}, {"LDBP_BWD_MODE": "0"}, {"LDBP_BWD_MODE": "1", "LDBP_REV3": "1"},
                                 {"LDBP_BWD_MODE": "1", "LDBP_REV4": "1"}, {"LDBP_BWD_MODE": "1", "LDBP_REV4": "0"},
                                 {"LDBP_BWD_MODE": "1", "LDBP_OVERLAP": "3"}, {"LDBP_BWD_MODE": "1", "LDBP_REV2": "1"}])
def test_repeated_runs_bitwise_identical(P, monkeypatch, env):
    """Race detector by repetition (compute-sanitizer is closed on this GPU pool): 12 repeated
    loss_grad calls of a store-all-sized problem, on two streams, must agree bit for bit — the
    mbarrier split barriers, ring buffers, cp.async windows and the fixed-order reductions leave
    no room for nondeterminism; a race would show as differing low bits.  Every schedule option."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("LDBP_STORE_ALL_MIN_SAMPLES", "0")
    B, n, M, T = 24, 16384, 10, 9
    x = dev(li.gaussian_blocks(61, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(61, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(61, M, T, True)
    ht, gt = dev(taps), dev(gamma, np.float32)
    ref = P.ldbp_loss_grad(x, tgt, ht, gt).cpu()
    s2 = torch.cuda.Stream()
    outs = []
    for i in range(12):
        st = s2 if i % 2 else torch.cuda.current_stream()
        s2.wait_stream(torch.cuda.current_stream())
        outs.append(P.ldbp_loss_grad(x, tgt, ht, gt, stream=st))
        torch.cuda.current_stream().wait_stream(s2)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o.cpu(), ref)
    r = O.loss_grad(r32(x.cpu().numpy()), r32(tgt.cpu().numpy()), r32(taps), r32(gamma), symmetric=True)
    assert abs(ref[0].item() - r[0]) <= OUT_TOL * r[0]
    assert rel(ref[1:].numpy(), r[1:]) <= GRAD_TOL


# ---- C1: the one-CTA fused training step (ldbp_tiny.cuh) ----
K_TINY = 9
TINY_CASES = [
    # (B, n, M, T, sym, masked)
    (4, 1024, 4, 3, True, False),    # BASELINE C1 exactly (4 segments per block, 16-CTA cluster)
    (2, 777, 3, 5, False, False),    # general taps, odd n: 3 uneven segments per block
    (3, 500, 5, 9, True, True),      # pruning mask
    (1, 5, 2, 5, True, False),       # n == T
    (2, 16, 6, 7, False, True),      # blocks shorter than the filter span (several wraps)
    (2, 64, 1, 1, True, False),      # T = 1, M = 1
    (1, 1000, 8, 15, True, False),   # Kh = 7 (the largest T)
    (11, 300, 3, 5, True, False),    # B > 8: 8-CTA cluster, CTAs 0-2 own two blocks
    (9, 64, 4, 3, False, True),      # ragged ownership, general taps, mask
    (8, 2048, 2, 9, True, False),    # whole blocks, 2 samples per thread
    (1, 4000, 3, 15, True, True),    # one block in 15 uneven segments (266/267), Kh = 7 halos over DSMEM
    (3, 300, 4, 7, False, False),    # blocks too short to split: whole blocks, C = 3
]


@pytest.mark.parametrize("B,n,M,T,sym,masked", TINY_CASES)
def test_tiny_fused_loss_grad_vs_oracle(P, monkeypatch, B, n, M, T, sym, masked):
    monkeypatch.setenv("LDBP_TINY", "2")  # whenever it fits (the default picks it for M <= 5)
    """Problems whose per-CTA activations fit shared memory run as ONE cluster launch (trace kind 9);
    parity with the oracle at the §8(c) tolerances, masked taps exactly 0, and agreement with the
    multi-launch segment schedule (LDBP_TINY=0) to the same tolerances."""
    x = li.gaussian_blocks(131, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(131, range(B), n, 1e-3, purpose="target")
    taps, gamma = model(131, M, T, sym)
    mask = None
    if masked:
        kh = (T - 1) // 2
        mask = np.ones((M, T), np.uint8)
        mask[0, [0, T - 1]] = 0
        if M > 2 and kh > 1:
            mask[2, [0, 1, T - 2, T - 1]] = 0
        taps = taps * mask
    mk = None if mask is None else torch.from_numpy(mask).cuda()
    with P.api.trace() as tr:
        buf = P.ldbp_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32), symmetric=sym, mask=mk)
        torch.cuda.synchronize()
    assert [r[0] for r in tr.records] == [K_TINY]
    assert P.launch_count(P.make_dims(B, n, M, T, sym), P._lib.OP_LOSS_GRAD) == 1
    buf = buf.cpu().numpy()
    ref = O.loss_grad(r32(x), r32(tgt), r32(taps), r32(gamma), mask=mask, symmetric=sym)
    assert abs(buf[0] - ref[0]) <= OUT_TOL * ref[0]
    for i in range(M):
        assert abs(buf[1 + i] - ref[1 + i]) <= GRAD_TOL * abs(ref[1 + i]) + 1e-12 * np.abs(ref[1:1 + M]).max(), i
    dt, rdt = buf[1 + M:].reshape(M, T, 2), ref[1 + M:].reshape(M, T, 2)
    for i in range(M):
        assert rel(dt[i], rdt[i]) <= GRAD_TOL, (i, rel(dt[i], rdt[i]))
    if masked:
        assert np.all(dt[mask == 0] == 0)
    monkeypatch.setenv("LDBP_TINY", "0")
    seg = P.ldbp_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32), symmetric=sym, mask=mk).cpu().numpy()
    assert abs(seg[0] - buf[0]) <= OUT_TOL * ref[0]
    assert rel(seg[1 + M:], buf[1 + M:]) <= GRAD_TOL


def test_tiny_fused_train_step(P):
    """ldbp_train_step at C1 is ONE launch (loss, gradient, fold, Adam); equal to the tiny
    loss_grad followed by ldbp_adam_update (same buffer bit for bit, fp64 master <= 1e-13), and its
    first Adam step equals the oracle's Adam on the oracle gradient to the gradient tolerance."""
    B, n, M, T = 4, 1024, 4, 3
    x = dev(li.gaussian_blocks(137, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(137, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(137, M, T, True)
    mask = np.ones((M, T), np.uint8)
    mask[1, [0, 2]] = 0
    gl = np.array([1, 0, 1, 1], np.uint8)
    taps = taps * mask
    s1 = P.TrainState.create(taps, gamma, mask=mask, gamma_learnable=gl)
    s2 = P.TrainState.create(taps, gamma, mask=mask, gamma_learnable=gl)
    for it in range(3):
        with P.api.trace() as tr:
            b1 = P.ldbp_train_step(s1, x, tgt)
            torch.cuda.synchronize()
        assert [r[0] for r in tr.records] == [K_TINY]
        b2 = P.ldbp_loss_grad(x, tgt, s2.taps, s2.gamma, mask=s2.mask)
        P.ldbp_adam_update(s2, b2, B * n)
        assert torch.equal(b1, b2), it
        assert rel(s1.master.cpu().numpy(), s2.master.cpu().numpy()) <= 1e-13
        assert torch.equal(s1.taps, s2.taps) or rel(s1.taps.cpu().numpy(), s2.taps.cpu().numpy()) <= 1e-7
    assert P.launch_count(P.make_dims(B, n, M, T), P._lib.OP_TRAIN_STEP) == 1
    # first step against the oracle
    s3 = P.TrainState.create(taps, gamma, mask=mask, gamma_learnable=gl)
    P.ldbp_train_step(s3, x, tgt)
    ref = O.loss_grad(r32(x.cpu().numpy()), r32(tgt.cpu().numpy()), r32(taps), r32(gamma), mask=mask, symmetric=True)
    th0 = O.pack_params(r32(taps), r32(gamma))
    th, _, _ = O.adam_update(ref, B * n, th0, np.zeros_like(th0), np.zeros_like(th0), 1, M, T, tap_mask=mask,
                             gamma_learnable=gl)
    # Adam's first step moves each parameter by ~lr sign(g): compare the step, not the value
    step, rstep = s3.master.cpu().numpy() - th0, th - th0
    assert rel(step, rstep) <= 1e-3


def test_tiny_fused_train_step_cuda_graph(P):
    """The fused C1 step captured in a CUDA graph (one kernel node) replays like eager calls."""
    B, n, M, T = 4, 1024, 4, 3
    x = dev(li.gaussian_blocks(139, range(B), n, 1e-3))
    tgt = dev(li.gaussian_blocks(139, range(B), n, 1e-3, purpose="target"))
    taps, gamma = model(139, M, T, True)
    eager = P.TrainState.create(taps, gamma)
    graphed = P.TrainState.create(taps, gamma)
    buf = torch.empty(1 + M + 2 * M * T, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        P.ldbp_loss_grad(x, tgt, graphed.taps, graphed.gamma, buf=buf)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    graphed.t = 0
    with torch.cuda.graph(g):
        P.ldbp_train_step(graphed, x, tgt, buf=buf)
    graphed.t = 0
    b_e = P.ldbp_train_step(eager, x, tgt)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(b_e, buf)
    assert torch.equal(eager.master, graphed.master)


# ---- wide filters: T = 17 .. 31 (1 <= T <= 31 compiled specialisations) ----
@pytest.mark.parametrize("T,sym", [(17, True), (17, False), (23, True), (31, True), (31, False)])
def test_wide_filters_forward_and_gradients(P, monkeypatch, T, sym):
    B, n, M = 3, 1500, 5
    x = li.gaussian_blocks(71, range(B), n, 1e-3)
    tgt = li.gaussian_blocks(71, range(B), n, 1e-3, purpose="target")
    taps, gamma = model(71, M, T, sym, scale=0.05)
    y = P.ldbp_forward(dev(x), dev(taps), dev(gamma, np.float32), symmetric=sym).cpu().numpy()
    ry = O.forward(r32(x), r32(taps), r32(gamma))
    for b in range(B):
        assert rel(y[b], ry[b]) <= OUT_TOL, (b, rel(y[b], ry[b]))
    ref = O.loss_grad(r32(x), r32(tgt), r32(taps), r32(gamma), symmetric=sym)
    for mode in ("0", "1"):  # checkpoint + segment backward, store-all + reverse
        set_mode(monkeypatch, mode, None)
        monkeypatch.setenv("LDBP_STORE_ALL_MIN_SAMPLES", "0")
        buf = P.ldbp_loss_grad(dev(x), dev(tgt), dev(taps), dev(gamma, np.float32), symmetric=sym).cpu().numpy()
        assert abs(buf[0] - ref[0]) <= OUT_TOL * ref[0], (mode, buf[0], ref[0])
        for i in range(M):
            assert abs(buf[1 + i] - ref[1 + i]) <= GRAD_TOL * abs(ref[1 + i]), (mode, i)
        dt, rdt = buf[1 + M:].reshape(M, T, 2), ref[1 + M:].reshape(M, T, 2)
        for i in range(M):
            assert rel(dt[i], rdt[i]) <= GRAD_TOL, (mode, i, rel(dt[i], rdt[i]))
