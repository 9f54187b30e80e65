"""Per-source-line instructions executed and stall samples of a single-kernel ncu report
(--import-source on, -lineinfo): python tools/ncu_lines.py REP [top]"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = ""
res = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name"):
        try:
            ie = int(r[7] or 0); smp = int(r[4] or 0)
        except ValueError:
            continue
        res.append((ie, smp, cur, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in res) or 1
tots = sum(x[1] for x in res) or 1
print(f"total instructions {tot/1e9:.3f} G, samples {tots}")
for ie, smp, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{ie/1e9:7.3f}G {100*ie/tot:5.1f}% {100*smp/tots:5.1f}%s  {f}:{ln}  {src}")
