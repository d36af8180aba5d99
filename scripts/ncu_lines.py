"""Per-source-line totals (warp instructions executed, stall samples) from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or not hdr or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ins = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    out.append((fname, int(r[0]), r[1][:70], ins, smp))
ti = sum(o[3] for o in out) or 1
ts = sum(o[4] for o in out) or 1
print(f"total warp instructions {ti}, samples {ts}")
for o in sorted(out, key=lambda o: -o[4])[:top]:
    print(f"{o[0]}:{o[1]:<5} ins {100*o[3]/ti:5.1f}% smp {100*o[4]/ts:5.1f}%  {o[2]}")
