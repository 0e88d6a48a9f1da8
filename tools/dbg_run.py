"""Debug helper: one DMA forward on cuda:0 -- dbg_run.py H N d [nvfp4|mxfp4|mxfp8] [check]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_03950_b200 as D  # noqa: E402

H, N, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
low = {"nvfp4": D.NVFP4, "mxfp4": D.MXFP4, "mxfp8": D.MXFP8_E4M3}[sys.argv[4] if len(sys.argv) > 4 else "nvfp4"]
torch.manual_seed(0)
q = torch.randn(1, H, N, d, device="cuda").bfloat16()
k = torch.randn(1, H, N, d, device="cuda").bfloat16()
v = torch.randn(1, H, N, d, device="cuda").bfloat16()
cfg = D.AttentionConfig(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=low)
o = D.DmaAttention(cfg)(q, k, v)
torch.cuda.synchronize()
msg = f"ok H={H} N={N} d={d} mean|o|={float(o.float().abs().mean()):.5f}"
if len(sys.argv) > 5:
    import numpy as np
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
    from oracle import mx_oracle as O
    lo = {D.NVFP4: O.NVFP4, D.MXFP4: O.MXFP4, D.MXFP8_E4M3: O.MXFP8_E4M3}[low]
    oc = O.Cfg(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format=lo)
    h = 0
    want = O.mixed_precision_attention(q[0, h].float().cpu().double().numpy(), k[0, h].float().cpu().double().numpy(),
                                       v[0, h].float().cpu().double().numpy(), oc, pv="mxfp8")
    got = o[0, h].float().cpu().double().numpy()
    ref = O.mixed_precision_attention(q[0, h].float().cpu().double().numpy(), k[0, h].float().cpu().double().numpy(),
                                      v[0, h].float().cpu().double().numpy(), oc)
    msg += f" rel-L2 vs emulation {np.linalg.norm(got - want) / np.linalg.norm(want):.3e}"
    msg += f" vs oracle {np.linalg.norm(got - ref) / np.linalg.norm(ref):.3e}"
print(msg)
