import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import ldbp_inputs as li
import paper_2010_14258_b200 as P
B, n, M, T, kap = 64, 16384, 2, 9, 20
x = torch.from_numpy(li.gaussian_blocks(1, range(B), n, 1e-3).astype(np.complex64)).cuda()
tg = torch.from_numpy(li.gaussian_blocks(1, range(B), n, 1e-3, purpose="target").astype(np.complex64)).cuda()
taps = torch.from_numpy(li.random_sym_taps(1, M, T, 0.1).astype(np.complex64)).cuda()
gam = torch.full((M,), -20.0, device="cuda")
eta = torch.full((M, 2 * kap + 1), 1.0 / (2 * kap + 1), device="cuda")
P.ldbp_essm_loss_grad(x, tg, taps, gam, eta)
torch.cuda.synchronize()
print("ok")
