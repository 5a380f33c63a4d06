"""Warp-stall samples per SASS instruction from an ncu report's source page
(first launch): totals by reason and the most-sampled instructions with
their neighbourhood.   python scripts/ncu_stalls.py report.ncu-rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", "regex:attn_mma"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) >= len(hdr):
        data.append(r)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {s: sum(int(r[ix[s]] or 0) for r in data) for s in stalls}
allsum = sum(tot.values())
print(f"{len(data)} instructions, {allsum} stall samples")
print("by reason:", ", ".join(f"{k[6:]} {100 * v / allsum:.1f}%" for v, k in sorted(((v, k) for k, v in tot.items()), reverse=True)[:10]))
recs = sorted(((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), n) for n, r in enumerate(data)), reverse=True)
for smp, n in recs[:n_top]:
    r = data[n]
    st = sorted(((int(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{n:6d} {smp:6d} {100 * smp / allsum:5.1f}% {r[ix['Source']].strip()[:64]:64s} {st}")
