"""Hot spots of an ncu report by warp-stall samples (source page, CUDA lines
with their SASS).   python scripts/ncu_hot.py REPORT [N]
Prints the top CUDA lines (file:line, share of samples, the two largest
stall reasons) and the top SASS instructions."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
lines = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
text = {}
sass = []
cur_line = None
hdr = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur_line = (fname, r[0])
        text[cur_line] = r[1].strip()
    try:
        smp = int(r[4])
    except ValueError:
        continue
    if r[2]:
        sass.append((smp, r[3].strip(), cur_line))
    lines[cur_line] += smp
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
            try:
                reasons[cur_line][h[6:]] += int(r[i])
            except ValueError:
                pass
tot = sum(s for s, _, _ in sass) or 1
print(f"total samples {tot}")
print("-- CUDA lines")
for (f, ln), smp in lines.most_common(n):
    top = ", ".join(f"{k} {100 * v / max(smp, 1):.0f}%" for k, v in reasons[(f, ln)].most_common(2) if v)
    print(f"{100 * smp / tot:5.1f}%  {f}:{ln:5s} {text.get((f, ln), '')[:70]:70s} [{top}]")
print("-- SASS")
for smp, s, cl in sorted(sass, key=lambda x: -x[0])[:n]:
    print(f"{100 * smp / tot:5.1f}%  {s[:70]:70s} {cl[0]}:{cl[1]}")
