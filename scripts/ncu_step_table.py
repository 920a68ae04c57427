"""Per-kernel durations of the last step in an ncu launch list (--metrics gpu__time_duration.sum --csv):
python scripts/ncu_step_table.py launches.csv [kernels_per_step]"""
import csv
import re
import sys


def short(n):
    m = re.search(r"(Epi\w+(?:<[^>]*>)?)", n)
    if "gemm_sm100_kernel" in n and m:
        mode = re.search(r"gemm_sm100_kernel<(\d+), (\d+)", n)
        return f"gemm<{mode.group(1)},{mode.group(2)}> {m.group(1)}"
    return re.sub(r"\(.*", "", n).replace("void ", "")[:60]


def main(path, per_step=None):
    rows = list(csv.reader(open(path)))
    hdr, L = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"])
                L.append((short(d["Kernel Name"]), v / 1000.0 if d.get("Metric Unit") == "ns" else v))
    # tamoe kernels only (skip torch fills etc.)
    L = [x for x in L if not x[0].startswith(("at::", "vectorized", "elementwise", "unrolled"))]
    n = int(per_step) if per_step else len(L)
    step = L[-n:]
    tot = sum(v for _, v in step)
    for name, v in step:
        print(f"{v:9.2f} us  {100 * v / tot:5.1f}%  {name}")
    print(f"{tot:9.2f} us  total ({len(step)} launches)")


if __name__ == "__main__":
    main(*sys.argv[1:])
