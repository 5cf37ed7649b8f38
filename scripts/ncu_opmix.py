"""Instruction mix of one ncu report's kernel by SASS opcode (read here, no GPU)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
mix = collections.Counter()
samples = collections.Counter()
tot = 0
for r in rows[1:]:
    try:
        n = int(r[ix["Instructions Executed"]])
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except (ValueError, IndexError):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    mix[op] += n
    samples[op] += smp
    tot += n
print(f"total warp-instructions {tot:.3e}")
for op, n in mix.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:12s} {n:.3e} {100 * n / tot:5.1f}%  stall-samples {samples[op]}")
