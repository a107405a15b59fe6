"""Aggregate ncu warp-stall samples per CUDA source line.
ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv
python tools/ncu_lines.py X.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
out = []
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        samp = int(r[4])
        ninst = int(r[7]) if r[7] not in ("-", "") else 0
    except (ValueError, IndexError):
        continue
    stalls = {}
    for k, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and k < len(r):
            try:
                v = int(r[k])
            except ValueError:
                continue
            if v:
                stalls[h[6:]] = v
    out.append((samp, fname, r[0], r[1][:90], ninst, stalls))
tot = sum(o[0] for o in out) or 1
out.sort(key=lambda o: -o[0])
print(f"total samples {tot}")
for s, f, ln, src, ni, st in out[:top]:
    st = ", ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{100*s/tot:5.1f}% {f}:{ln:>5} inst={ni:<8} {src:<90} [{st}]")
