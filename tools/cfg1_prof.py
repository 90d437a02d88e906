"""Config 1 (cnn3, one 28x28 image, N = 2^13): eager forwards inside the NVTX range `cfg1`
for an ncu launch list (how many launches one single-image request is, and their device time)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2402_01296_b200 as BCN
import synthetic
from paper_2402_01296_b200.archive import TensorArchive
from paper_2402_01296_b200.network import DecomposedInput

bundle = BCN.get("cnn3")
w = TensorArchive(synthetic.weights_for(synthetic.tensor_shapes(bundle), 0.1, seed=1))
sens, full = synthetic.cfg1_inputs(1, seed=0)
dec = [DecomposedInput(sens[0], full[0], (7, 7, 14, 14))]
ctx = BCN.make_context(8192, BCN.required_levels(bundle) + 1, 2.0 ** 50)
for it in range(4):
    torch.cuda.synchronize()
    if it == 3:
        torch.cuda.nvtx.range_push("cfg1")
    BCN.forward_bicrypto(bundle.bi, dec, w, ctx, strategy="hw").decrypt_logits()
    torch.cuda.synchronize()
    if it == 3:
        torch.cuda.nvtx.range_pop()
print("done")
