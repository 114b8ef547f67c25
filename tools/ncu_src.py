"""Summarise an ncu --page source --csv (--print-source sass) export: samples
per region of the SASS listing with the dominant stall reasons.
Usage: python tools/ncu_src.py export.csv [region_size]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
size = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, data = rows[1], rows[2:]
isrc, iss, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iss] or 0) for r in data)
print(f"{len(data)} instructions, {tot} samples, {sum(int(r[iex] or 0) for r in data)} warp-instructions executed")
for b in range(0, len(data), size):
    blk = data[b:b + size]
    s = sum(int(r[iss] or 0) for r in blk)
    if s < tot * 0.01:
        continue
    reasons = {hdr[i][6:]: sum(int(r[i] or 0) for r in blk) for i in stalls}
    top = sorted(reasons.items(), key=lambda kv: -kv[1])[:3]
    rep = max(blk, key=lambda r: int(r[iss] or 0))
    print(f"{b:5d}-{b + size - 1:5d} {100 * s / tot:5.1f}%  " + " ".join(f"{k}={v}" for k, v in top) +
          f"   | {rep[isrc].strip()[:60]}")
