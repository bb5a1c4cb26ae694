"""Small end-to-end workload for compute-sanitizer (test layer T5):
c0-shaped block prefill + decode (GEMV), a batched decode step (split-K GEMM and
the row-wise finalize), the persistent stack decode, centred-norm quant and a
c1-shaped BitLinear on both contraction paths.  Exits 0 when it ran through.
python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

L.load()
cfg = synth.CONFIGS["c0"]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda")
B, T = 2, 128
x = synth.hidden((B, T + 2, cfg.d), synth.generator(1, "cuda"), "f32", device="cuda")
h = st.new_state(B)
st.prefill(x[:, :T].contiguous(), h)
for t in range(T, T + 2):
    st.decode(x[:, t].contiguous(), h)
st.decode(x[:, T].contiguous(), h, persistent=True)
# batched decode: split-K GEMM + epilogue, then the row-wise finalize variant
xb = synth.hidden((24, cfg.d), synth.generator(2, "cuda"), "f32", device="cuda")
hb = st.new_state(24)
st.decode(xb, hb)
L.tern_set_batched_fin(True)
st.decode(xb, hb)
L.tern_set_batched_fin(False)
# centred norm stack (prefill + decode)
stc = model.Stack.random(cfg, device="cuda", gen_device="cuda", norm=L.TERN_NORM_CENTERED)
hc = stc.new_state(B)
stc.prefill(x[:, :T].contiguous(), hc)
stc.decode(x[:, T].contiguous(), hc)
# c1-shaped BitLinear (bf16, K=2048 -> N=5632): GEMV (m=1) and tensor-core (m=256) paths
W = synth.latent_matrix(5632, 2048, synth.generator(3, "cuda"), device="cuda")
pw = model.PackedWeight([W])
for m in (1, 256):
    xm = synth.hidden((m, 2048), synth.generator(4, "cuda"), "bf16", device="cuda")
    y = torch.empty((m, 5632), dtype=torch.bfloat16, device="cuda")
    L.bitlinear_fwd(xm, pw.struct, y)
torch.cuda.synchronize()
print("sanitize workload ok")
