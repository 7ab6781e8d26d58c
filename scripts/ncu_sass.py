"""Per-SASS-instruction rows of an `ncu --page source --print-source cuda,sass`
CSV export: for a given file:line, list each SASS instruction with its executed
count (to see which inlined copies of a source line run how often)."""
import csv, sys
path, want = sys.argv[1], sys.argv[2]  # e.g. fw_walk.cu:76
wf, wl = want.split(":")
fname = None; cur = None; out = []
for r in csv.reader(open(path)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0]:
        cur = (fname, r[0]); continue
    if cur == (wf, wl) and r[2] not in ("...", "-"):
        try: out.append((int(r[7]), r[2], r[3].strip()))
        except ValueError: pass
tot = sum(o[0] for o in out)
print(f"{want}: {len(out)} SASS instr, {tot:.4e} executed")
for n, addr, s in sorted(out, reverse=True)[: int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{n:14d} {addr} {s}")
