"""Summarise an ncu report: key metrics, stall reasons, hot instruction blocks."""
import collections, csv, subprocess, sys

rep = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof_slide.ncu-rep"
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ("Duration", "Executed Instructions |", "Issue Slots", "Eligible Warps", "Active Warps Per",
        "Registers", "Grid Size", "Block Size", "Achieved Active Warps", "DRAM Throughput", "Block Limit")
for line in det.splitlines():
    f = line.split('","')
    if len(f) > 4:
        name = f[-3] if len(f) >= 3 else ""
        txt = " | ".join(x.strip('"') for x in f[-4:])
        if any(k.rstrip(" |") == name or k in txt for k in keys):
            print(txt[:150])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
for h, v in zip(rows[0], rows[2]):
    if h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
             "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
             "lts__t_sector_hit_rate.pct", "gpu__time_duration.sum"):
        print(f"{h:70s} {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
st = collections.Counter()
for r in data:
    for c in cols:
        st[c] += int(r[ix[c]] or 0)
s = sum(st.values()) or 1
print("stalls:", [(c[6:], round(100 * v / s, 1)) for c, v in st.most_common(8)])
by = collections.defaultdict(list)
for r in data:
    by[int(r[ix["Instructions Executed"]] or 0)].append(r)
for n, rs in sorted(by.items(), key=lambda kv: -kv[0] * len(kv[1]))[:9]:
    ops = collections.Counter(); samp = collections.Counter()
    for r in rs:
        op = r[ix["Source"]].split(); op = op[1] if op[0].startswith("@") else op[0]
        ops[op.split(".")[0]] += 1
        for c in cols:
            samp[c[6:]] += int(r[ix[c]] or 0)
    print(f"{n:>8} x {len(rs):>4} = {100*n*len(rs)/tot:5.1f}% stall {100*sum(samp.values())//s:3d}% "
          f"{samp.most_common(3)} {ops.most_common(7)}")
print("total warp-instructions", tot)
