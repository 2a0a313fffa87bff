"""Per-source-line executed warp instructions and stall samples from an ncu report
(--page source, cuda+sass interleaved).  usage: lines_prof.py REPORT [top_n]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
inst = collections.Counter()
samp = collections.Counter()
text = {}
cur = None
fname = ""
hdr = None
for r in csv.reader(src.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:70]
        continue
    ie = r[hdr["Instructions Executed"]]
    sm = r[hdr["Warp Stall Sampling (All Samples)"]]
    inst[cur] += int(ie) if ie.isdigit() else 0
    samp[cur] += int(sm) if sm.isdigit() else 0
tot = sum(inst.values()) or 1
ts = sum(samp.values()) or 1
print(f"total warp instructions {tot}, samples {ts}")
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k[0]}:{k[1]:4d} {100*v/tot:5.1f}% inst {100*samp[k]/ts:5.1f}% samp  {text.get(k, '')}")
