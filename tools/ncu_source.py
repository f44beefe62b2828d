"""Top SASS lines by warp-stall samples with their dominant stall reasons (dev tool)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
f = lambda r, h: float(r[idx[h]] or 0)
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    s = f(r, "Warp Stall Sampling (All Samples)")
    top = sorted(((f(r, h), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}%  {r[idx['Source']][:58]:58s} " + " ".join(f"{h}={v:.0f}" for v, h in top if v))
