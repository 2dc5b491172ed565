"""Top source lines by warp-stall samples from an ncu report (dev tool).

usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, out = "?", None, {}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) >= 5 and r[0].isdigit() and r[2] == "-":  # source-line rows
        try:
            v = int(r[4])
        except ValueError:
            continue
        if v:
            out[(fname, int(r[0]))] = (v, r[1].strip()[:100])
tot = sum(v[0] for v in out.values()) or 1
for (f, ln), (v, src) in sorted(out.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{v:7d} {100 * v / tot:5.1f}%  {f}:{ln}  {src}")
