"""Forwards of the MoE layer at a given shape (world 1) for ncu captures of the gate kernels:
python tools/gate_profile.py T d E k [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2404_19429_b200 import lancet  # noqa: E402

T, d, E, k = (int(v) for v in sys.argv[1:5])
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
f = 256
sh = S.LayerShape(T=T, d=d, f=f, E=E, G=1, k=k, cf=1.25, n_chunks=1)
ins = S.gen_rank_inputs(3, 0, sh, beta=0.25, with_dy=False)
bf = torch.bfloat16
x = torch.from_numpy(ins["x"]).cuda().to(bf)
wg = torch.from_numpy(ins["wg"]).cuda()
w1 = torch.from_numpy(ins["w1"]).cuda().to(bf)
w2 = torch.from_numpy(ins["w2"]).cuda().to(bf)
ctx = lancet.Context(lancet.LayerConfig(d_model=d, d_ffn=f, n_experts=E, max_tokens=T, max_k=k))
for _ in range(steps):
    ctx.forward(x, wg, w1, w2, k, 1.25, 1)
torch.cuda.synchronize()
ctx.close()
print("ok")
