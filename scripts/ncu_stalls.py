"""Top stall sites (SASS) of the first kernel in an ncu report."""
import csv
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
ia, isrc = hdr.index('Address'), hdr.index('Source')
iss = hdr.index('Warp Stall Sampling (All Samples)')
tot = sum(float(r[iss] or 0) for r in data) or 1
top = sorted(data, key=lambda r: -float(r[iss] or 0))[:n]
for r in sorted(top, key=lambda r: int(r[ia], 16)):
    print(r[ia][-5:], f"{100 * float(r[iss]) / tot:5.1f}%", r[isrc][:100])
