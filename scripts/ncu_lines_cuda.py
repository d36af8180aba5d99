"""Per-CUDA-source-line stall samples and warp instructions from an ncu report
(`--page source --print-source=cuda,sass`), optionally bucketed by sim.cu line ranges:

    python scripts/ncu_lines_cuda.py gpurun_out/crit.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, recs, hdr = None, [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or not r[0] or hdr is None or len(r) < 8:
        continue
    try:
        samples, inst = int(r[4]), int(r[7])
    except ValueError:
        continue
    recs.append((fname, int(r[0]), r[1].strip()[:70], samples, inst))
ts = sum(x[3] for x in recs) or 1
ti = sum(x[4] for x in recs) or 1
print(f"total samples {ts}, warp instructions {ti}")
for f, ln, src, s, i in sorted(recs, key=lambda x: -x[3])[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst  {f}:{ln}  {src}")
