"""Summarise an ncu source-page CSV (SASS): stall reasons and the hottest instructions.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv; python tools/ncu_hot.py X.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = rows[1]; data = rows[2:]
reasons = [x for x in h if x.startswith('stall_') and 'Not Issued' not in x]
idx = {r: h.index(r) for r in reasons}
tot = {r: sum(int(d[idx[r]] or 0) for d in data) for r in reasons}
T = sum(tot.values())
print({r[6:]: round(100 * v / T, 1) for r, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
iss = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
print("total samples", T, "warp insts", sum(int(d[ex] or 0) for d in data))
top = sorted(range(len(data)), key=lambda i: -int(data[i][iss] or 0))[:top_n]
for i in sorted(top):
    d = data[i]
    rs = {r[6:]: int(d[idx[r]]) for r in reasons if int(d[idx[r]] or 0) > 0.15 * int(d[iss])}
    print(i, d[iss], d[1][:70], rs)
