"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv --print-source sass`
(optionally cuda,sass for line correlation). Usage: ncu_hot.py file.csv [topN]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
ci = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_")]
tot = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
print("total samples", tot)
agg = {}
for r in body:
    for s in stalls:
        agg[s] = agg.get(s, 0) + int(r[ci[s]] or 0)
print("stall totals:", ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
top = sorted(body, key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    n = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    main = sorted(((int(r[ci[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{100*n/tot:5.1f}% {r[0][-5:]} {r[1].strip()[:60]:60s} {main}")
