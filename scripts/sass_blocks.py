"""Basic-block view of an ncu --page source --print-source sass CSV: consecutive SASS lines with
the same executed count are one block; prints per block its size, executed count, share of all
warp-instructions and stall samples, plus the first opcodes (scripts/, analysis only)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def num(x):
    try: return float(x.replace(',', ''))
    except ValueError: return 0.0
minshare = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
tot_i = sum(num(d['Instructions Executed']) for d in data)
tot_s = sum(num(d['Warp Stall Sampling (All Samples)']) for d in data)
blocks = []
for idx, d in enumerate(data):
    c = num(d['Instructions Executed'])
    if blocks and blocks[-1][1] == c:
        blocks[-1][2].append(idx)
    else:
        blocks.append([idx, c, [idx]])
print('total warp-instr %.4e  samples %d' % (tot_i, tot_s))
print('%6s %5s %10s %6s %6s  %s' % ('idx', 'len', 'exec', 'inst%', 'smp%', 'ops'))
for start, c, idxs in blocks:
    share = 100 * c * len(idxs) / tot_i
    smp = sum(num(data[i]['Warp Stall Sampling (All Samples)']) for i in idxs)
    if share < minshare and 100 * smp / tot_s < minshare:
        continue
    ops = ' '.join(data[i]['Source'].split()[1 if data[i]['Source'].startswith('@') else 0].split('.')[0] for i in idxs[:14])
    print('%6d %5d %10.3e %6.2f %6.2f  %s' % (start, len(idxs), c, share, 100 * smp / tot_s, ops))
