"""Top SASS instructions by warp-stall samples of one kernel in an ncu report.
usage: python tools/ncu_src.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
h = rows[hi]
A = h.index("Address"); S = h.index("Source"); W = h.index("Warp Stall Sampling (All Samples)"); I = h.index("Instructions Executed")
# first kernel only (a report with several kernels repeats the header)
body = []
for r in rows[hi + 1:]:
    if "Source" in r or (len(r) > 0 and r[0] == "Kernel Name"):
        break
    if len(r) > max(W, I): body.append(r)
def f(x):
    try: return float(x or 0)
    except ValueError: return 0.0
tot = sum(f(r[W]) for r in body)
tins = sum(f(r[I]) for r in body)
print(f"samples {tot:.0f}  warp-instructions {tins:.0f}")
res = sorted(((f(r[W]), k, r) for k, r in enumerate(body)), reverse=True)[:top]
for w, k, r in sorted(res, key=lambda x: x[1]):
    print(f"{100*w/tot:5.1f}%  #{k:<5d} inst={r[I]:>9s}  {r[S][:90]}")
