"""Top source lines of an ncu report by warp-stall samples, with the main
stall reasons.  python tools/ncu_hot.py REPORT [N] [cuda|sass]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
view = sys.argv[3] if len(sys.argv) > 3 else "cuda"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                     capture_output=True, text=True).stdout
rows, hdr, fname, total = [], None, "", 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Address"):
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    total += s
    reasons = sorted(((int(d[k] or 0), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k),
                     reverse=True)[:3]
    rows.append((s, fname, r[0], d["Source"].strip()[:70], reasons))
rows.sort(reverse=True)
print("total samples", total)
for s, f, ln, src, rs in rows[:n]:
    print(f"{s:7d} {100.0 * s / max(total, 1):5.1f}% {f}:{ln:6s} {src:70s} {' '.join(f'{k}={v}' for v, k in rs if v)}")
