"""bench.py's CPU legs (cpu_baseline, --impl reference): the row-split multi-thread
harness computes the same step as the oracle's own stack (O.stack_f64)."""
import numpy as np

import oracle as O
import synth


def test_threaded_oracle_step_matches_stack_f64():
    import bench
    cfg = dict(layers=3, hidden=256, heads=4, kv_heads=2, head_dim=64, ffn=384)
    d, H, G, hd, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
    W = (O.quantize(35, 64, np.concatenate([synth.weight(0, "q", H * hd, d, d), synth.weight(0, "k", G * hd, d, d),
                                            synth.weight(0, "v", G * hd, d, d)])),
         O.quantize(35, 64, synth.weight(0, "o", d, H * hd, d)),
         O.quantize(35, 64, np.concatenate([synth.weight(0, "gate", Fd, d, d), synth.weight(0, "up", Fd, d, d)])),
         O.quantize(35, 64, synth.weight(0, "down", d, Fd, d)))
    h = synth.activations(2, d)
    L = cfg["layers"]
    ref, _ = O.stack_f64(dict(cfg, qtype=35, block=64), [W[0]] * L, [W[1]] * L, [W[2]] * L, [W[3]] * L, h)
    for threads in (1, 3, 8):
        got = bench.stack_rows_threaded(cfg, W, h, threads)
        # activations enter each threaded matmul as fp32 (ref_matmul_f64's input type)
        assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-6
