"""Top CUDA source lines by warp-stall samples from an ncu report (needs -lineinfo builds).
usage: python tools/ncu_lines.py report.ncu-rep [kernel-substring] [N]"""
import csv
import io
import subprocess
import sys


def main(rep, ksub="", n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    func, hdr, res = None, None, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or (ksub and ksub not in (func or "")):
            continue
        try:
            si = hdr.index("Warp Stall Sampling (All Samples)")
            s = int(r[si] or 0)
        except (ValueError, IndexError):
            continue
        if r[2] != "-":  # sass rows repeat under their source line
            continue
        key = (func[:40], r[0], r[1].strip()[:110])
        res[key] = res.get(key, 0) + s
    tot = sum(res.values()) or 1
    for (f, ln, src), s in sorted(res.items(), key=lambda x: -x[1])[:n]:
        print(f"{100 * s / tot:5.1f}% {s:6d}  L{ln:>4}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 25)
