"""Per-CUDA-source-line instruction and stall-sample attribution from an
`ncu --page source --csv --print-source cuda,sass` export."""
import csv, sys
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = []
fname = None
tot_i = tot_s = 0
with open(path) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            inst = int(r[7]); samp = int(r[4])
        except (ValueError, IndexError):
            continue
        tot_i += inst; tot_s += samp
        rows.append((inst, samp, fname, r[0], r[1].strip()[:90]))
print(f"total warp inst {tot_i:.4e}, samples {tot_s}")
for inst, samp, fn, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*inst/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% samp  {fn}:{ln}  {src}")
