"""Per-region stall breakdown from an ncu source page: sums stall reasons over SASS address ranges."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]
ai, si = h.index("Address"), h.index("Source")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = [h.index(x) for x in reasons]
tot = collections.Counter()
for r in data:
    for n, i in zip(reasons, ri):
        tot[n] += float(r[i] or 0)
T = sum(tot.values())
print("overall:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in tot.most_common(10)))
# top instructions with their dominant reasons
wi = h.index("Warp Stall Sampling (All Samples)")
top = sorted(range(len(data)), key=lambda i: -float(data[i][wi] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for i in sorted(top):
    r = data[i]
    rs = sorted(((float(r[j] or 0), n[6:]) for n, j in zip(reasons, ri)), reverse=True)[:3]
    print(f"{i:5d} {100*float(r[wi])/T:5.2f}%  {r[si].strip()[:60]:60s} " + " ".join(f"{n}:{100*v/T:.2f}" for v, n in rs if v > 0))
