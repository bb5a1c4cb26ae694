"""One bitlinear_bwd call at the c2 o-projection shape (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

m, k, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 1024, 1024)))
L.load()
W = synth.latent_matrix(n, k, synth.generator(1)).cuda()
pw = model.PackedWeight([W])
x = torch.randn(m, k, device="cuda")
dO = torch.randn(m, n, device="cuda")
dX, dW, db = torch.empty_like(x), torch.empty(n, k, device="cuda"), torch.empty(n, device="cuda")
for _ in range(2):
    L.bitlinear_bwd(x, pw.struct, dO, dX, dW, db)
torch.cuda.synchronize()
