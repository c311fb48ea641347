"""paper_2010_14258_b200 — B200-native hot path of learned digital backpropagation (LDBP).

Häger & Pfister, "Physics-Based Deep Learning for Fiber-Optic Communication Systems",
arXiv:2010.14258.  The compute lives in libldbp.so (hand-written sm_100a CUDA behind the C ABI
of include/ldbp.h); this package is the thin binding plus host-side helpers.
"""
from .api import (  # noqa: F401
    AdamConfig,
    TrainState,
    Workspace,
    launch_count,
    ldbp_adam_update,
    ldbp_backward,
    ldbp_essm_forward,
    ldbp_essm_loss_grad,
    ldbp_forward,
    ldbp_loss_grad,
    ldbp_loss_grad_state,
    ldbp_rx_exact_loss_grad,
    ldbp_rx_exact_train_grad,
    ldbp_rx_loss_grad,
    ldbp_rx_train_grad,
    ldbp_ssfm_link,
    ldbp_train_step,
    ldbp_tx_waveform,
    make_dims,
    workspace_bytes,
)
from ._lib import LIB_PATH, LdbpError  # noqa: F401
