"""Per-source-line hotspots of an ncu report (ncu -i REP --page source --print-source cuda,sass):
stall samples and excess shared wavefronts summed over the SASS of each CUDA line.
Usage: ncu_lines.py REP [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
samples = collections.Counter()
excess = collections.Counter()
text = {}
fname = "?"
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:90]
    if cur is None:
        continue
    def f(k):
        try:
            return float(r[hdr[k]].replace(",", ""))
        except (KeyError, ValueError):
            return 0.0
    samples[cur] += f("Warp Stall Sampling (All Samples)")
    excess[cur] += f("L1 Wavefronts Shared Excessive")
tot = sum(samples.values()) or 1
print(f"{rep}: {tot:.0f} stall samples")
for k, v in samples.most_common(top):
    print(f"{100 * v / tot:5.1f}%  excess_shared {excess[k]:>12.0f}  {k[0]}:{k[1]}  {text.get(k, '')}")
print("top excess shared wavefronts:")
for k, v in excess.most_common(8):
    print(f"{v:>12.0f}  {k[0]}:{k[1]}  {text.get(k, '')}")
