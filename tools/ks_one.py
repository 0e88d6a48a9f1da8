"""One small forward with a forced KV split (for ncu): python tools/ks_one.py H N mode"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_03950_b200 as D
from paper_2604_03950_b200 import _lib
H, N, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
L = _lib.lib()
L.dma_attention_set_kv_split(mode)
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=D.NVFP4)
q, k, v = (torch.randn(1, H, N, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
fwd = D.DmaAttention(cfg)
a, out = fwd.prepare(q, k, v)
sp = _lib.stream_ptr(torch.cuda.current_stream())
for _ in range(3):
    _lib.check(L.dma_attention_fwd(a, sp), "fwd")
torch.cuda.synchronize()
print("ns", L.dma_attention_kv_split(a))
