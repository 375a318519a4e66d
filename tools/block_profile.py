"""A few block forwards (+ backwards with BWD=1) at BASELINE configs[3] per GPU (one-rank group)
for ncu / compute-sanitizer: python tools/block_profile.py [n_chunks] [steps]   (env E, BWD)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2404_19429_b200 import block as B, lancet  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
bwd = os.environ.get("BWD", "0") == "1"
sh = S.BlockShape(n_seq=int(os.environ.get("NSEQ", "8")), seq_len=1024, d=2048, n_heads=16, f=8192,
                  E=int(os.environ.get("E", "32")), G=1, k=1, cf=1.25, n_chunks=n)
ins = S.gen_block_rank_inputs(2031, 0, sh, beta=0.25, with_dy=False)
bf = torch.bfloat16
p = {k: torch.from_numpy(ins[k]).cuda().to(torch.float32 if k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "wg") else bf)
     for k in B.PARAMS}
x = torch.from_numpy(ins["x"]).cuda().to(bf)
moe = lancet.LayerConfig(d_model=sh.d, d_ffn=sh.f, n_experts=sh.E, max_tokens=sh.T, max_k=1, max_chunks=8)
blk = B.Block(B.BlockConfig(moe, n_heads=sh.n_heads, seq_len=sh.seq_len, max_capacity_factor=1.25))
out = torch.empty_like(x)
dout = torch.randn(x.shape, device="cuda").to(bf)
for _ in range(steps):
    blk.forward(x, p, 1, 1.25, n, out=out)
    if bwd:
        g = blk.backward(dout)
    torch.cuda.synchronize()
blk.close()
print("ok")
