#!/usr/bin/env python
"""bench.py — decode tokens/s and HBM GB/s of the 3.5-bit qGEMV stack on B200.

Workload (BASELINE.json configs[1]): Llama-2-7B-shaped linear stack (32 layers,
d 4096, F 11008), Q3H_B64 (3.5-bit, 4.0 bits/weight), batch-1 decode.  A step
is one if_run_stack call: all 32 layers (RMSNorm -> fused qkv qGEMV ->
single-position GQA -> o qGEMV + residual -> RMSNorm -> fused gate/up qGEMV ->
SiLU*u -> down qGEMV + residual).  Weights are synthetic (device generator),
3.24 GB packed, far larger than the 126 MB L2, so every step streams them from
HBM (no flush needed).  The step is replayed from a CUDA graph.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--model 7b]
  python bench.py --impl reference ...     (the CPU oracle)

N > 1 (torchrun, one process per GPU): the same stack partitioned by layer
(default: each stage one persistent engine launch, hand-off through the
peer-memory communicator) or --strategy tensor|hybrid (per-layer kernels +
peer-memory merges); value = tokens/s of the job, time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s & HBM GB/s (% of peak) for 3.5-bit qGEMV stack at 1/2/4/8 B200"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), float(mp.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle, as it stands
# ---------------------------------------------------------------------------
def _oracle_layer(model: str):
    """Layer 0 of the stack, quantized by the oracle from the host generator."""
    import numpy as np

    import oracle as O
    import synth

    cfg = synth.LLAMA[model]
    d, H, G, hd, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
    l = 0
    wqkv = O.quantize(35, 64, np.concatenate([synth.weight(l, "q", H * hd, d, d), synth.weight(l, "k", G * hd, d, d),
                                              synth.weight(l, "v", G * hd, d, d)]))
    wo = O.quantize(35, 64, synth.weight(l, "o", d, H * hd, d))
    wgu = O.quantize(35, 64, np.concatenate([synth.weight(l, "gate", Fd, d, d), synth.weight(l, "up", Fd, d, d)]))
    wd = O.quantize(35, 64, synth.weight(l, "down", d, Fd, d))
    return cfg, ([wqkv], [wo], [wgu], [wd])


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    import synth

    cfg, W = _oracle_layer(args.model)
    L = cfg["layers"]
    h = synth.activations(args.batch, cfg["hidden"])
    shape1 = dict(cfg, layers=1, qtype=35, block=64)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.stack_f64(shape1, *W, h)
        t1 = time.perf_counter()
        if i >= args.warmup:
            times.append(t1 - t0)
    t_layer = sum(times) / len(times)
    value = args.batch / (t_layer * L)
    sample = f"one of the {L} layers of the {args.model} stack per step (fp64 oracle, 1 thread), time x{L}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_layer * L * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"llama2-{args.model}-stack q3h_b64 decode b={args.batch}",
                   "model": f"llama2-{args.model}-shaped", "global_batch": args.batch, "seq_len": 1,
                   "parallelism": "single", "scheme": "Q3H_B64 (4.0 bits/weight)"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(model: str, batch: int, budget_s: float = 10.0):
    """The oracle timed on a bounded sample of the workload: layer 0 of the
    stack, repeated for ~budget_s, extrapolated to all layers."""
    import oracle as O
    import synth

    cfg, W = _oracle_layer(model)
    L = cfg["layers"]
    h = synth.activations(batch, cfg["hidden"])
    shape1 = dict(cfg, layers=1, qtype=35, block=64)
    reps, t_total = 0, 0.0
    while t_total < budget_s:
        t0 = time.perf_counter()
        O.stack_f64(shape1, *W, h)
        t_total += time.perf_counter() - t0
        reps += 1
    value = batch / (t_total / reps * L)
    return {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle",
            "sample": f"layer 0 of the {model} stack x{reps} runs ({t_total:.1f} s), fp64 oracle single-threaded, "
                      f"time per layer x{L}"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2401_08294_b200 as F
    import synth
    from paper_2401_08294_b200.model import Stack

    ws, rank, local = dist_env()
    # IFB_BENCH_SHARE_GPU=1: every rank on cuda:0, gloo plumbing (a functional check
    # of the N-rank path on a 1-GPU box; its timing is not a scaling number)
    share = os.environ.get("IFB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    hbm_peak, bf16_peak, peak_kind = peaks()
    cfg = synth.LLAMA[args.model]
    s = F.scheme("Q3H", 64)
    shape = F.stack_shape(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"], s)
    if ws == 1:
        plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
        strategy = "single"
    elif args.strategy == "layer":
        plan = F.if_plan_partition(F.IF_BY_LAYER, shape, ws)
        strategy = f"pp{ws}"
    elif args.strategy == "hybrid":
        st = args.stages or 2
        plan = F.if_plan_partition(F.IF_HYBRID, shape, ws, st, ws // st)
        strategy = f"pp{st}xtp{ws // st}"
    else:
        plan = F.if_plan_partition(F.IF_BY_TENSOR, shape, ws)
        strategy = f"tp{ws}"
    B = args.batch
    stk = Stack(cfg, s, plan, rank, dev)
    comm = None
    if ws > 1:
        comm = F.Comm(plan, rank, max(B, 64), cfg["hidden"])
        comm.exchange()
    d = cfg["hidden"]
    h_in = torch.from_numpy(synth.activations(B, d)).to(dev)
    h_out = torch.empty_like(h_in)
    wsb = torch.zeros(F.if_stack_workspace_bytes(shape, plan, rank, B, F.IF_DECODE), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)

    def step():
        F.if_run_stack(shape, plan, rank, comm, stk.arr, h_in, B, F.IF_DECODE, h_out, None, wsb, stream)

    # launches per step (our kernels), counted on one eager step
    with torch.cuda.stream(stream):
        F.if_launch_count(reset=True)
        step()
        launches_per_step = F.if_launch_count(reset=True)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        step()  # warm (attributes set before capture)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=stream):
            step()
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        graph.replay()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                graph.replay()
            e1.record(stream)
        e1.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    tok_s = B * args.steps / (ms / 1e3)  # tokens of the job (one stream of B tokens per step)
    total_bytes = stack_bytes_total(cfg, s)
    gbs = total_bytes / (ms_per_step / 1e3) / 1e9  # whole-job weight bytes streamed per second
    rank_bytes = stk.weight_bytes()
    stack_gbs_rank = rank_bytes / (ms_per_step / 1e3) / 1e9

    # ---- e2e through the public API: pinned host h_in -> device -> stack -> host h_out
    h_host = torch.from_numpy(synth.activations(B, d)).pin_memory()
    o_host = torch.empty_like(h_host).pin_memory()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            h_in.copy_(h_host, non_blocking=True)
            graph.replay()
            o_host.copy_(h_out, non_blocking=True)
        stream.synchronize()
        f0.record(stream)
        for _ in range(args.steps):
            h_in.copy_(h_host, non_blocking=True)
            graph.replay()
            o_host.copy_(h_out, non_blocking=True)
        f1.record(stream)
    f1.synchronize()
    ms_e2e = f0.elapsed_time(f1)
    if dist:
        t = torch.tensor([ms_e2e], device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e = {"value": B * args.steps / (ms_e2e / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": B * d * 4,
           "d2h_bytes_per_step": B * d * 4}

    # ---- roofline of the dominant kernel.  For batch-1 Q3H the whole step is ONE
    #      launch of the persistent decode kernel (decode_mk: 128 fused-dequant
    #      GEMV phases + glue), so its average launch duration is the step time
    #      measured above on the launching stream (the graph adds only a 16 KB
    #      device copy and a 512 B memset around it).  Algorithmic bytes per
    #      launch = the packed weights of the rank's layers (0.5 B/weight).
    launches_mk = launches_per_step
    roof = {"kernel": "decode_mk (persistent whole-stack decode, 1 launch/step)" if launches_mk == 1 else
            "qgemv (per-layer kernels)", "bound": "hbm", "achieved": stack_gbs_rank,
            "peak": hbm_peak, "unit": "GB/s", "frac": stack_gbs_rank / hbm_peak,
            "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
            "traffic": None, "avg_launch_us": ms_per_step * 1e3 / max(1, launches_mk),
            "algorithmic_bytes_per_launch": rank_bytes // max(1, launches_mk),
            "algorithmic_bytes": "packed weight bytes (0.5 B/weight incl. two fp16 per 64-block)"}
    prof_path = os.path.join(ROOT, "profiles", "decode_mk_traffic.json")
    if os.path.exists(prof_path):
        try:
            with open(prof_path) as f:
                roof["traffic"] = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            pass

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (counter-based Irwin-Hall weights sigma=1/sqrt(d), activations sigma=1)",
            "config": {"workload": f"llama2-{args.model}-stack q3h_b64 decode b={B}", "model": f"llama2-{args.model}-shaped",
                       "global_batch": B, "seq_len": 1, "parallelism": strategy, "scheme": "Q3H_B64 (4.0 bits/weight)",
                       "weight_bytes_per_step": total_bytes,
                       "l2": f"inputs larger than L2 ({total_bytes / 1e9:.2f} GB of weights per step vs 126 MB L2)"},
            "hbm_gbs": gbs, "hbm_frac_of_measured": gbs / hbm_peak / ws,
            "hbm_frac_of_nominal_8tbs": gbs / 8000.0 / ws,
            "roofline": roof, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
    if comm:
        comm.destroy()
    if dist:
        dist.destroy_process_group()
    return line


def stack_bytes_total(cfg, s):
    import paper_2401_08294_b200 as F
    d, H, G, hd, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
    per = (F.if_packed_bytes(s, (H + 2 * G) * hd, d) + F.if_packed_bytes(s, d, H * hd) +
           F.if_packed_bytes(s, 2 * Fd, d) + F.if_packed_bytes(s, d, Fd))
    return per * cfg["layers"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--model", default="7b", choices=["7b", "13b", "70b"])
    # N > 1 default: by layer -- every stage runs the persistent decode engine; by
    # tensor / hybrid run the per-layer kernels + peer-memory merges
    ap.add_argument("--strategy", default="layer", choices=["tensor", "layer", "hybrid"])
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    line = run_ours(args)
    ws, rank, _ = dist_env()
    if rank == 0 and line is not None:
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.model, args.batch)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
