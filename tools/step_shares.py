"""Per-kernel shares of the timed HMult+Relin steps in an ncu launch list of
`bench.py` taken with --nvtx --nvtx-include "timed/" and the metrics
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum.
The list starts with the timed steps (each begins with tensor_d2_kernel);
later timed legs (rotate, rescale, e2e, NTT roofline) are ignored.

    python tools/step_shares.py launches.csv [steps] [out.txt]
"""
import csv
import re
import sys
from collections import OrderedDict, defaultdict

_SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
          "s": 1e6, "second": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)(<[^(]*>)?", name)
    return (m.group(0) if m else name)[:72]


def main(path, steps="2", out=None):
    steps = int(steps)
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, d = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID",
                                               "Metric Unit"))
    launches = OrderedDict()
    for r in d:
        launches.setdefault(r[ii], {"name": r[ki]})[r[mi]] = \
            float(r[vi].replace(",", "")) * _SCALE.get(r[ui], 1.0)
    agg, cnt, byt = defaultdict(float), defaultdict(int), defaultdict(float)
    items = list(launches.values())
    names = [short(x["name"]) for x in items]
    heads = [i for i, n in enumerate(names) if n.startswith(("tensor_d2_kernel", "tensor_kernel"))]
    per = heads[1] - heads[0]  # kernels per step (the steps are back to back)
    tot = 0.0
    for it, n in zip(items[heads[0]:heads[0] + steps * per], names[heads[0]:heads[0] + steps * per]):
        t = it.get("gpu__time_duration.sum", 0.0)
        agg[n] += t
        cnt[n] += 1
        byt[n] += it.get("dram__bytes_read.sum", 0.0) + it.get("dram__bytes_write.sum", 0.0)
        tot += t
    lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache and",
             f"# serialised: compare SHARES).  {steps} timed HMult+Relin steps of bench.py:"]
    for n, t in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"{n:72s} launches={cnt[n]:3d} total_us={t:9.1f} share={100 * t / tot:5.1f}%"
                     f" dram_GB={byt[n] / 1e9:6.2f}")
    lines.append(f"TOTAL {tot:.1f} us for {steps} steps -> {tot / steps:.1f} us/step")
    text = "\n".join(lines) + "\n"
    print(text)
    if out:
        open(out, "w").write(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
