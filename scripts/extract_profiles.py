"""Turn the round's ncu reports (gpurun_out/*.ncu-rep) into committed summaries under
profiles/: per-kernel key metrics CSV + the traffic JSON bench.py reads."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.min.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.max.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, vals = rows[0], rows[1], rows[2]
    return {k: (v, u) for k, u, v in zip(h, units, vals)}, h


def main(tag, reps):
    summary = {}
    for name in reps:
        rep = os.path.join(ROOT, "gpurun_out", name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        d, h = raw(rep)
        row = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
        for k in KEYS:
            if k in d:
                row[k] = d[k][0] + (f" {d[k][1]}" if d[k][1] else "")
        summary[name] = row
        with open(os.path.join(OUT, f"{tag}_{name}_metrics.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["metric", "value", "unit"])
            for k in h:
                if k in d and d[k][0] != "":
                    w.writerow([k, d[k][0], d[k][1]])
    with open(os.path.join(OUT, f"{tag}_ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    g = summary.get("group_int_m16")
    if g:
        def mb(s):
            v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else ""
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return float(v) * scale
        t = mb(g["dram__bytes_read.sum"]) + mb(g["dram__bytes_write.sum"])
        with open(os.path.join(OUT, f"{tag}_traffic.json"), "w") as f:
            json.dump({"grouped_layer_m16_bytes_per_launch": t,
                       "source": f"ncu --set full, profiles/{tag}_group_int_m16_metrics.csv "
                                 "(dram__bytes_read.sum + dram__bytes_write.sum)"}, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    names = (["group_int_m16", "group_float_m16", "pf_sp_gu_m2048", "pf_group_m2048",
              "pf_float_gu_m2048"] if tag == "r02b" else
             ["group_int_m16", "group_float_m16", "group_int_m32", "group_float_m32", "group_int_m64",
              "pf_sp_gu_m2048", "pf_group_m2048", "pf_float_gu_m2048", "pf_int8192_gu_m2048"]
             if tag == "r02d" else
             ["group_int_m16", "group_float_m16", "group_int_m1", "pf_int_m2048", "pf_float_m2048"])
    main(tag, names)
