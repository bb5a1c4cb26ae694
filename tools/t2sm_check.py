import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from paper_2406_02528_b200 import _lib as L, model as M, synth
L.load()
L.tern_set_gemm_2sm(True)
for (m, k, n, dt) in [(512, 1024, 1024, "f32"), (4096, 2048, 5632, "bf16"), (300, 256, 192, "f32")]:
    g = synth.generator(1)
    W = synth.latent_matrix(n, k, g)
    pw = M.PackedWeight([W.cuda()])
    t, mw = O.ternarize(W.numpy())
    x = synth.hidden((m, k), g, dt)
    y = torch.empty((m, n), dtype=synth.torch_dtype(dt), device="cuda")
    L.bitlinear_fwd(x.cuda(), pw.struct, y)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.random.default_rng(0).choice(m, 16, replace=False), [0, m - 1, min(255, m-1), min(256, m-1)]]))
    ref = O.bitlinear(x.float().numpy()[rows], t, mw, bf16=(dt == "bf16"))
    got = y.float().cpu().numpy()[rows]
    print(m, k, n, dt, "2sm exact:", np.array_equal(got, ref), float(np.abs(got - ref).max()))
