"""Top CUDA source lines by warp-stall samples from
`ncu -i X --page source --csv --print-source cuda,sass` (one section per file).
Usage: ncu_lines.py file.csv[.gz] [topN]"""
import csv, gzip, sys
path = sys.argv[1]
fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(fh))
out, fname, hdr = [], "?", None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        width = len(r)
        stalls = [h for h in r if h.startswith("stall_")]
        continue
    if hdr and r and r[0] and len(r) == width:
        n = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        st = sorted(((int(r[hdr[s]] or 0), s[6:]) for s in stalls if r[hdr[s]] not in ("", "-")), reverse=True)[:3]
        out.append((n, f"{fname}:{r[0]}", r[1].strip()[:80], st))
tot = sum(o[0] for o in out)
print("total samples", tot)
for n, loc, src, st in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*n/tot:5.1f}% {loc:22s} {src:80s} {st}")
