"""Calibrate the partition cost model (if_cost_model, Q29) on this B200 and
record the auto-planner's choices -> profiles/r2_cost_calibration.json.

Measured here (1 GPU): the batch-1 decode step of the 7B / 13B / 70B stacks
(bench.py, one persistent launch per token).  Fit per token:
    t_step = L * t_fixed + L * layer_bytes / bw          (least squares over 3 models)
Not measurable on a 1-GPU pool: the NVLink merge and hand-off latencies.  They are
taken from the measured NVLink constants of /opt/skills/guides/B300_MICROARCH.md
(peer load 1834 cycles at the 1.965 GHz SM clock = 0.93 us; peer bandwidth 775 GB/s):
    t_merge(g) = 2 * 0.93 us + (g - 1) * bytes / 775 GB/s  (one-shot peer all-reduce:
                 stores to the peers + flag, then one remote read; B = 1 rows)
    t_hop      = 0.93 us + bytes / 775 GB/s
    python scripts/calibrate_cost.py [--steps 30]
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2401_08294_b200 as F  # noqa: E402
import synth  # noqa: E402

NVL_LAT = 1834 / 1.965e9
NVL_BW = 775e9


def layer_bytes(cfg):
    s = F.scheme(35, 64)
    d, H, G, hd, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
    return sum(F.if_packed_bytes(s, N, K) for N, K in [((H + 2 * G) * hd, d), (d, H * hd), (2 * Fd, d), (d, Fd)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_cost_calibration.json"))
    a = ap.parse_args()
    meas = {}
    for m in ("7b", "13b", "70b"):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--model", m, "--steps", str(a.steps),
                            "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=1500)
        line = json.loads(r.stdout.strip().splitlines()[-1])
        cfg = synth.LLAMA[m]
        meas[m] = dict(ms_per_step=line["ms_per_step"], tok_s=line["value"], layers=cfg["layers"],
                       layer_bytes=layer_bytes(cfg), frac=line["roofline"]["frac"])
        print(m, meas[m], flush=True)
    A = np.array([[v["layers"], v["layers"] * v["layer_bytes"]] for v in meas.values()], np.float64)
    y = np.array([v["ms_per_step"] * 1e-3 for v in meas.values()])
    (t_fixed, inv_bw), *_ = np.linalg.lstsq(A, y, rcond=None)
    bw = 1.0 / inv_bw
    fit = {m: float(A[i] @ [t_fixed, inv_bw] * 1e3) for i, m in enumerate(meas)}
    out = dict(measured=meas, fit=dict(t_fixed_s=float(t_fixed), bw_bytes_s=float(bw), predicted_ms=fit))
    plans = {}
    for m in ("13b", "70b"):
        cfg = synth.LLAMA[m]
        shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")],
                              F.scheme(35, 64))
        rowbytes = 4 * cfg["hidden"]
        tm = [0.0] + [2 * NVL_LAT + (g - 1) * rowbytes / NVL_BW for g in range(1, 9)]
        cm = F.cost_model(t_fixed, bw, tm, NVL_LAT + rowbytes / NVL_BW)
        for devices in (1, 2, 4, 8):
            for obj in ("decode", "throughput"):
                p, dec, thr = F.if_plan_auto(obj, shape, devices, cm, micro_batches=devices)
                plans[f"{m} {devices}gpu {obj}"] = dict(stages=p.stages, groups=p.groups, decode_tok_s=dec,
                                                        throughput_tok_s=thr)
            grid = {}
            for g in range(1, devices + 1):
                if devices % g == 0:
                    try:
                        grid[f"{devices // g}x{g}"] = F.if_cost_estimate(shape, devices // g, g, cm, devices)
                    except F.IFError:
                        pass
            plans[f"{m} {devices}gpu all grids (stages x groups: decode, throughput)"] = grid
    out["nvlink"] = dict(source="B300_MICROARCH.md NVLink table (measured on 8x B300 NV18; not measurable on the "
                         "1-GPU pool)", peer_latency_s=NVL_LAT, peer_bw_bytes_s=NVL_BW)
    out["plans"] = plans
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
