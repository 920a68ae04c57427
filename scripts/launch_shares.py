"""Summarise an ncu launch list (gpu__time_duration.sum) of bench.py into per-kernel-family shares of one step."""
import csv
import json
import sys


def fam(n):
    if "gemm_sm100_kernel<2," in n:
        return "gate logits GEMM (tcgen05)"
    if "EpiSwap" in n:
        return "expert grouped GEMM fwd/dgrad (tcgen05, swap-AB)"
    if "EpiWgrad" in n:
        return "expert grouped GEMM wgrad (tcgen05)"
    for k in ["route_logits", "EpiGateDw", "EpiGateDx", "route_scan", "route_bucket", "route_capacity", "route_permute",
              "combine_loss", "gate_dz", "dwg_reduce", "ep_plan"]:
        if k in n:
            return k
    return None


def main(path, out):
    rows = list(csv.reader(open(path)))
    hdr, L = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                L.append((d["Kernel Name"], float(d["Metric Value"])))
    ours = [(n, t) for n, t in L if fam(n)]
    gates = [i for i, (n, t) in enumerate(ours) if fam(n).startswith("gate logits")]
    step = ours[gates[-1]:]  # last (warm) step
    tot = sum(t for _, t in step)
    agg = {}
    for n, t in step:
        agg[fam(n)] = agg.get(fam(n), 0.0) + t
    res = {"source": path, "launches_in_step": len(step), "step_total_us": round(tot / 1e3, 1),
           "us": {k: round(v / 1e3, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])},
           "share": {k: round(v / tot, 4) for k, v in sorted(agg.items(), key=lambda x: -x[1])},
           "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised launches; "
                   "compare shares, not absolute times"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
