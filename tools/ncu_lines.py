"""Per-source-line totals (instructions executed, stall samples) from an ncu report's
correlated cuda+sass source view: python tools/ncu_lines.py REPORT.ncu-rep [TOP]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = "?"
cur = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":  # a source line row
        cur = (fname, int(r[0]), r[1].strip()[:70])
        continue
    try:
        s = int(r[4]); e = int(r[7])
    except ValueError:
        continue
    if cur:
        a = agg.setdefault(cur, [0, 0])
        a[0] += s; a[1] += e
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts} instructions {te}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/ts:5.1f}% samp {100*v[1]/te:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
