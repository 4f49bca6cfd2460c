"""Per-kernel SASS instruction mix and stall samples from an ncu report's
source page (ncu --set full --import-source on).

    python tools/sass_mix.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, top=25):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    blocks = txt.split('"Kernel Name"')
    for blk in blocks[1:]:
        lines = ('"Kernel Name"' + blk).splitlines()
        name = lines[0].split(",", 1)[1][:110]
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr = rows[0]
        iS, iE, iT = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        ops = defaultdict(lambda: [0, 0])
        stalls = defaultdict(float)
        tot_i = tot_s = 0
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            src = r[iS].strip()
            if not src or src.startswith("."):
                continue
            op = src.split()[0]
            if op.startswith("@"):
                op = src.split()[1]
            op = op.split(".")[0]
            try:
                n, s = int(r[iE]), int(r[iT])
            except ValueError:
                continue
            ops[op][0] += n
            ops[op][1] += s
            tot_i += n
            tot_s += s
            for i, h in stall_cols:
                try:
                    stalls[h] += float(r[i])
                except ValueError:
                    pass
        print(f"== {name}\n   warp-instructions {tot_i}, stall samples {tot_s}")
        for op, (n, s) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:top]:
            print(f"   {op:10s} {n:12d} {100.0 * n / max(tot_i, 1):5.1f}%  samples {100.0 * s / max(tot_s, 1):5.1f}%")
        st = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("   stalls:", ", ".join(f"{h[6:]}={100.0 * v / max(tot_s, 1):.1f}%" for h, v in st))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
