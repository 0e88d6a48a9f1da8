"""Case tables shared by the golden generator and the tests (no reference import)."""

ATTN_CASES = [
    # name, Lq, Lk, d, dv, seed, cfg kwargs
    ("default_c_256_d64", 256, 256, 64, 64, 11, dict()),
    ("mxfp4_t128_256_d64", 256, 256, 64, 64, 12,
     dict(tile_m=128, tile_n=128, diag_window=128, sink_window=128, low_format="mxfp4")),
    ("ragged_200_d64", 200, 200, 64, 64, 13, dict(diag_window=64, sink_window=64)),
    ("nvfp4_t128_384_d128", 384, 384, 128, 128, 14,
     dict(tile_m=128, tile_n=128, diag_window=128, sink_window=128)),
    ("noncausal_192x256_d64", 192, 256, 64, 64, 15,
     dict(causal=False, diag_window=128, sink_window=64)),
    ("noncausal_t128_256_d128", 256, 256, 128, 128, 16,
     dict(tile_m=128, tile_n=128, causal=False, diag_window=256, sink_window=128)),
    ("identity_256_d64", 256, 256, 64, 64, 17, dict(low_format=None, high_format=None)),
    ("lowNone_256_d64", 256, 256, 64, 64, 18, dict(low_format=None, diag_window=64)),
    ("low8_256_d64", 256, 256, 64, 64, 19, dict(low_format="mxfp8_e4m3")),
    ("block_256_d64", 256, 256, 64, 64, 20, dict(granularity="block", diag_window=64)),
    ("tensor_256_d64", 256, 256, 64, 64, 21, dict(granularity="tensor", sink_window=64)),
    ("e5m2_t128_256_d128", 256, 256, 128, 128, 22,
     dict(tile_m=128, tile_n=128, high_format="mxfp8_e5m2", low_format="mxfp4", diag_window=0)),
    ("dv32_c_128_d64", 128, 128, 64, 32, 23, dict(tile_m=32, tile_n=32, diag_window=32)),
]

# (name, L, d, seed, AttentionConfig kwargs) for mixed_precision_scores
SCORE_CASES = [
    ("causal_nvfp4_token", 256, 64, 41, dict(tile_m=64, tile_n=64, diag_window=64, sink_window=64, causal=True)),
    ("causal_mxfp4_block", 192, 64, 43, dict(tile_m=64, tile_n=64, diag_window=128, sink_window=0, causal=True,
                                             low_format="mxfp4", granularity="block")),
    ("noncausal_nvfp4_tensor", 160, 32, 45, dict(tile_m=32, tile_n=32, diag_window=64, sink_window=32,
                                                 causal=False, granularity="tensor")),
    ("causal_identity_low", 128, 64, 47, dict(tile_m=32, tile_n=32, diag_window=32, sink_window=0, causal=True,
                                              low_format=None)),
]
