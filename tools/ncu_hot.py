"""Summarise an ncu report's source page: top CUDA lines by warp-stall
samples (with the dominant stall reasons).  python tools/ncu_hot.py rep [n] [inst]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hdr_i]
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[2] == "-"]
    if "Warp Stall Sampling (All Samples)" not in hdr:
        print("columns:", hdr[:10])
        return
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
    stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    key = si
    if len(sys.argv) > 3 and sys.argv[3] == "inst" and ii is not None:
        key = ii
        print(f"total warp instructions {sum(f(r[ii]) for r in data):.0f}")
    total = sum(f(r[si]) for r in data)
    data.sort(key=lambda r: -f(r[key]))
    print(f"total samples {total:.0f}")
    for r in data[:top]:
        s = f(r[si])
        if s == 0 and key == si:
            break
        reasons = sorted(((f(r[k]), hdr[k][6:]) for k in stall_cols), reverse=True)[:3]
        rs = ", ".join(f"{n}:{v / s:.0%}" for v, n in reasons if v > 0)
        ins = f(r[ii]) if ii is not None else 0
        print(f"{s / max(total, 1):6.1%} L{r[0]:>5} inst={ins:>10.0f} [{rs}] {r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
