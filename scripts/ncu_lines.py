"""Per-source-line instruction counts and stall samples from an ncu report's cuda,sass source
view (run here on the CPU side):  python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys

def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr, lines = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and r[0] != "":
            d = dict(zip(hdr[4:], r[4:]))
            try:
                lines.append((fname, int(r[0]), r[1].strip()[:70], int(d["Instructions Executed"] or 0),
                              int(d["Warp Stall Sampling (All Samples)"] or 0)))
            except (KeyError, ValueError):
                pass
    tot_i = sum(l[3] for l in lines) or 1
    tot_s = sum(l[4] for l in lines) or 1
    print(f"total warp instructions {tot_i:.3e}, stall samples {tot_s}")
    for l in sorted(lines, key=lambda l: -l[3])[:top]:
        print(f"{l[0]}:{l[1]:<5} {100 * l[3] / tot_i:5.1f}% inst {100 * l[4] / tot_s:5.1f}% smp  {l[2]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
