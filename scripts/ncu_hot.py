"""Summarise an ncu --page source --print-source sass CSV: top instructions by
stall samples, with the dominant stall reasons (read here, no GPU)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
tot = 0
for r in rows[1:]:
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except (ValueError, IndexError):
        continue
    tot += s
    data.append((s, r))
data.sort(key=lambda t: -t[0])
print("total samples", tot)
for s, r in data[:top]:
    reasons = sorted(((int(r[ix[h]]), h[6:]) for h in stalls if r[ix[h]].isdigit()), reverse=True)[:3]
    print(f"{s:7d} {100*s/tot:5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} "
          + " ".join(f"{n}:{v}" for v, n in reasons if v))
