"""Executed warp-instructions per CUDA line of an ncu report, normalised per
CTA and per coordinate.   python scripts/ncu_instr.py REPORT CTAS COORDS [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, ctas, coords = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, cur, hdr = "?", None, None
cnt, txt = collections.Counter(), {}
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or r[0] == "Function Name" or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, r[0])
        txt[cur] = r[1].strip()
    if r[2]:
        try:
            cnt[cur] += int(r[hdr["Instructions Executed"]])
        except (ValueError, KeyError):
            pass
tot = sum(cnt.values())
print(f"warp-instructions per CTA per coordinate: {tot / ctas / coords:.0f}")
for k, v in cnt.most_common(n):
    print(f"{v / ctas / coords:8.1f}  {k[0]}:{k[1]:5s} {txt.get(k, '')[:90]}")
