"""Warp-instruction share of line ranges of one source file, from an ncu report's cuda,sass
source view.   python scripts/ncu_regions.py report.ncu-rep file.cu name:lo-hi [name:lo-hi ...]"""
import csv, subprocess, sys

def main(path, fname_want, regions, per=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr, agg, tot = None, None, {}, 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]; continue
        if r[0] == "Line No":
            hdr = r; continue
        if hdr and r[0].isdigit():
            d = dict(zip(hdr[4:], r[4:]))
            try:
                n = int(d.get("Instructions Executed") or 0)
            except ValueError:
                continue
            tot += n
            ln, key = int(r[0]), "other:" + str(fname)
            if fname == fname_want:
                key = "rest of " + fname
                for name, lo, hi in regions:
                    if lo <= ln <= hi:
                        key = name; break
            agg[key] = agg.get(key, 0) + n
    print(f"total warp instructions {tot:.4e}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{k:32s} {100 * v / tot:5.1f}%" + (f"  {v / per:9.0f} per unit" if per else ""))

if __name__ == "__main__":
    regs = []
    per = None
    for a in sys.argv[3:]:
        if a.startswith("per="):
            per = float(a[4:]); continue
        n, rng = a.split(":")
        lo, hi = rng.split("-")
        regs.append((n, int(lo), int(hi)))
    main(sys.argv[1], sys.argv[2], regs, per)
