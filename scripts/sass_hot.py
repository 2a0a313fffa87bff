"""Summarise an ncu --page source --print-source sass CSV: instructions executed and stall
samples per SASS region (scripts/, analysis only)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def num(x):
    try: return float(x.replace(',', ''))
    except: return 0.0
tot_i = sum(num(d['Instructions Executed']) for d in data)
tot_s = sum(num(d['Warp Stall Sampling (All Samples)']) for d in data)
print('total warp-instr %.3e  samples %d' % (tot_i, tot_s))
top = sorted(data, key=lambda d: -num(d['Instructions Executed']))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for d in top:
    print('%-8s %10.3e %6d  %s' % (d['Address'], num(d['Instructions Executed']), num(d['Warp Stall Sampling (All Samples)']), d['Source'][:90]))
