import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2604_03950_b200 as D
torch.manual_seed(0)
H, N, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
q = torch.randn(1, H, N, d, device="cuda").bfloat16(); k = torch.randn(1, H, N, d, device="cuda").bfloat16(); v = torch.randn(1, H, N, d, device="cuda").bfloat16()
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=D.NVFP4)
o = D.DmaAttention(cfg)(q, k, v)
torch.cuda.synchronize()
print("ok", H, N, d, float(o.float().abs().mean()))
