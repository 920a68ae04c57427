"""Summarise an `ncu --set full` capture of one step's tcgen05 GEMM launches (scripts/profile_round.sh) into
profiles/: the raw per-launch metrics CSV and the per-GEMM DRAM traffic JSON that bench.py's roofline cites.

  python scripts/ncu_summary.py gpurun_out/r01_gemms.ncu-rep profiles/r01_ncu_full_gemms.csv profiles/r01_gemm_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__time_duration.sum", "launch__cluster_dim_x", "launch__grid_size", "launch__registers_per_thread",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
ORDER = ["gate logits", "fwd1", "fwd2", "gate dW", "dgrad2", "wgrad2", "wgrad1", "dgrad1", "gate dX"]
EXPERT = ["fwd1", "fwd2", "dgrad2", "wgrad2", "wgrad1", "dgrad1"]


def scale(v, unit):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)


def main(rep, out_csv, out_json):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    with open(out_csv, "w") as f:
        f.write(txt)
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    launches = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    assert len(launches) == len(ORDER), f"expected the {len(ORDER)} GEMM launches of one step, got {len(launches)}"
    u = dict(zip(hdr, units))
    per = {}
    for name, d in zip(ORDER, launches):
        per[name] = {
            "kernel": d["Kernel Name"][:80],
            "us": scale(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"]),
            "dram_read": scale(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]),
            "dram_write": scale(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]),
            "dram_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
            "tensor_pct": float(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]),
            "lts_pct": float(d["lts__throughput.avg.pct_of_peak_sustained_elapsed"]),
        }
    traffic = sum(per[n]["dram_read"] + per[n]["dram_write"] for n in EXPERT) / len(EXPERT)
    res = {"kernel": "expert grouped GEMM family (6 launches/step)", "traffic_bytes_per_launch": traffic,
           "source": rep.split("/")[-1] + " (ncu --set full --clock-control none, scripts/profile_round.sh)",
           "per_launch": {n: per[n]["dram_read"] + per[n]["dram_write"] for n in EXPERT},
           "per_kernel": per, "launch_order": ORDER}
    with open(out_json, "w") as f:
        json.dump(res, f, indent=1)
    for n in ORDER:
        p = per[n]
        print(f"{n:12s} {p['us']:8.1f} us  dram {p['dram_pct']:5.1f}%  tensor {p['tensor_pct']:5.1f}%  "
              f"lts {p['lts_pct']:5.1f}%  traffic {(p['dram_read'] + p['dram_write']) / 1e6:8.1f} MB")


if __name__ == "__main__":
    main(*sys.argv[1:4])
