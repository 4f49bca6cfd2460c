"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list of
`bench.py --steps 2 --warmup 1`: per-kernel totals over the two timed steps.

    python tools/launch_shares.py gpurun_out/bench_launches.csv [out.txt]
"""

import csv
import re
import sys
from collections import OrderedDict, defaultdict


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)(<[^(]*>)?", name)
    return (m.group(0) if m else name)[:72]


def main(path: str, out: str | None = None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = OrderedDict()
    for r in data:
        launches.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    items = list(launches.values())
    names = [short(x["name"]) for x in items]
    tens = [i for i, n in enumerate(names) if n.startswith("tensor_")]
    # the list is either a whole run (warm-up + 2 timed steps + later phases:
    # take the last two steps before the first non-step kernel) or an
    # nvtx-filtered "timed/" list (the 2 timed batched steps come first)
    nvtx_first = "--nvtx-first" in sys.argv
    start = tens[0] if nvtx_first else (tens[-2] if len(tens) >= 2 else 0)
    end = len(items)
    for i in range(start + 1, len(items)):
        if names[i].startswith("tensor_") and i > tens[-1]:
            end = i
            break
    # stop at the first non key-switch kernel after the last step (e2e / NTT phases)
    agg, cnt, byt = defaultdict(float), defaultdict(int), defaultdict(float)
    tot = 0.0
    step_kernels = ("tensor_", "ntt_tiles", "ntt_tma", "ntt_fused", "modup", "ks_inner", "moddown")
    seen_tensor = 0
    for it, n in zip(items[start:], names[start:]):
        if n.startswith("tensor_"):
            seen_tensor += 1
            if seen_tensor > 2:
                break
        if not n.startswith(step_kernels):
            break
        t = it.get("gpu__time_duration.sum", 0.0) / 1e3
        agg[n] += t
        cnt[n] += 1
        if seen_tensor == 2 and n.startswith("moddown_finish"):
            break  # end of the last timed step (the NTT roofline legs follow)
        byt[n] += it.get("dram__bytes_read.sum", 0.0) + it.get("dram__bytes_write.sum", 0.0)
        tot += t
    lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache and",
             "# serialised: compare SHARES).  Two timed HMult+Relin steps (batch 8 each):"]
    for n, t in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"{n:72s} launches={cnt[n]:3d} total_us={t:9.1f} share={100 * t / tot:5.1f}%"
                     f" dram_GB={byt[n] / 1e9:6.2f}")
    lines.append(f"TOTAL {tot:.1f} us for 2 steps -> {tot / 2:.1f} us/step")
    text = "\n".join(lines) + "\n"
    print(text)
    if out:
        open(out, "w").write(text)


if __name__ == "__main__":
    main(*[a for a in sys.argv[1:] if not a.startswith("--")])
