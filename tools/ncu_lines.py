"""Top source lines of an ncu report by warp-stall samples: python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:   # one kernel (regex on its name)
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res, hdr, tot = None, [], None, 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 4 and r[0] not in ("",) and r[0].isdigit():
        s = int(r[4]) if r[4].isdigit() else 0
        tot += s
        res.append((s, fname, r[0], r[1].strip()[:110]))
res.sort(reverse=True)
print("total samples", tot)
for s, f, ln, src in res[:N]:
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {f}:{ln}  {src}")
