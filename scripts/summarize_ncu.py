"""Summarise ncu reports into profiles/ (text + json)."""
import csv, io, json, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, rows = r[0], r[1], r[2:]
    return [{k: (v, unit) for k, unit, v in zip(h, u, row)} for row in rows]


def main(rep, name, out_txt, out_json=None, bytes_alg=None):
    rows = raw(rep)
    lines = [f"# ncu --set full summary: {name} ({rep})"]
    res = {}
    for i, row in enumerate(rows):
        kn = row.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## launch {i}: {kn[:120]}")
        for k in WANT:
            if k in row:
                v, unit = row[k]
                lines.append(f"  {k:70s} {v} {unit}")
                try:
                    res[k] = float(v.replace(",", ""))
                except ValueError:
                    pass
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if "dram__bytes_read.sum" in rows[0] and "dram__bytes_write.sum" in rows[0]:
        rv, ru = rows[0]["dram__bytes_read.sum"]
        wv, wu = rows[0]["dram__bytes_write.sum"]
        tot = float(rv.replace(",", "")) * mult.get(ru, 1) + float(wv.replace(",", "")) * mult.get(wu, 1)
        lines.append(f"  dram bytes per launch (read+write): {tot:.4e}")
        if bytes_alg:
            lines.append(f"  algorithmic bytes per launch: {bytes_alg:.4e}  (traffic / algorithmic = {tot / bytes_alg:.3f})")
        res["dram_bytes_per_launch"] = tot
    open(out_txt, "w").write("\n".join(lines) + "\n")
    if out_json:
        json.dump({"report": rep, "dram_bytes_per_launch": res.get("dram_bytes_per_launch"),
                   "duration": res.get("gpu__time_duration.sum"), "metrics": res}, open(out_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 and sys.argv[4] != "-" else None,
         float(sys.argv[5]) if len(sys.argv) > 5 else None)
