"""Regenerate tests/golden/tune/candidates.json: tile candidate lists, padding and
tops_of from the UNMODIFIED reference (oracle/gen_tune_golden.cpp).  Run here,
where the reference tree exists:

    make -C oracle ref && python tests/golden/make_tune_golden.py
"""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "tests", "golden", "tune", "candidates.json")
os.makedirs(os.path.dirname(OUT), exist_ok=True)
data = json.loads(subprocess.run([os.path.join(ROOT, "oracle", "_ref", "gen_tune_golden")], check=True,
                                 capture_output=True, text=True).stdout)
import hashlib  # noqa: E402


def digest(cands):
    """sha256 of the candidate list in order, "BM,BN,BK,WM,WN,WK;" per tile"""
    return hashlib.sha256("".join("%d,%d,%d,%d,%d,%d;" % tuple(c) for c in cands).encode()).hexdigest()


out = []
for d in data:
    if "candidates" in d:
        c = d.pop("candidates")
        d.update(count=len(c), sha256=digest(c), first=c[0], last=c[-1])
    out.append(d)
with open(OUT, "w") as f:
    json.dump(out, f, separators=(",", ":"))
print("wrote", OUT, len(data) - 1, "cases")
