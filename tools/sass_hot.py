"""Stall samples of one kernel's SASS, summed over windows of W instructions
(ncu --set full --import-source on report).

    python tools/sass_hot.py report.ncu-rep KERNEL_INDEX [W] [--list]
"""
import csv
import io
import subprocess
import sys


def load(path, kidx):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    blk = txt.split('"Kernel Name"')[1 + kidx]
    lines = ('"Kernel Name"' + blk).splitlines()
    name = lines[0][:140]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    return name, hdr, [r for r in rows[1:] if len(r) == len(hdr)]


def main():
    path, kidx = sys.argv[1], int(sys.argv[2])
    W = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
    name, hdr, data = load(path, kidx)
    iS, iT, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    sc = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not" not in h]
    tot = sum(int(r[iT] or 0) for r in data)
    print(name, "samples", tot)
    if "--list" in sys.argv:
        for k, r in enumerate(data):
            s = int(r[iT] or 0)
            top = max(((float(r[i] or 0), h) for i, h in sc))
            print(f"{k:5d} {s:5d} {r[iE]:>9s} {r[iS].strip()[:64]:64s} {top[1]}={top[0]:.0f}")
        return
    for w0 in range(0, len(data), W):
        win = data[w0:w0 + W]
        s = sum(int(r[iT] or 0) for r in win)
        if s < 0.01 * tot:
            continue
        st = {}
        for r in win:
            for i, h in sc:
                st[h] = st.get(h, 0) + float(r[i] or 0)
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        ops = {}
        for r in win:
            op = r[iS].split()[0] if r[iS].split() else "?"
            if op.startswith("@") and len(r[iS].split()) > 1:
                op = r[iS].split()[1]
            ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
        mix = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:5])
        print(f"{w0:5d}-{w0 + W - 1:5d} {100.0 * s / tot:5.1f}%  "
              + " ".join(f"{h}={100.0 * v / tot:.1f}" for h, v in top) + f"   [{mix}]")


if __name__ == "__main__":
    main()
