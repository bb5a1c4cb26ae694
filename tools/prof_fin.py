"""ncu driver: a few c4 B=128 decode steps with the row-wise finalize (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_02528_b200 import _lib as L, model, synth
L.load()
L.tern_set_batched_fin(True)
cfg = synth.CONFIGS["c4"]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=1)
x = synth.hidden((128, cfg.d), synth.generator(1, "cuda"), cfg.dtype, device="cuda")
h = st.new_state(128)
for _ in range(3):
    st.decode(x, h)
torch.cuda.synchronize()
print("ok")
