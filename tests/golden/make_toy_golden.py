"""Regenerate tests/golden/toy/toy.json: the reference toy block's seeded weights,
input, forward_fp and forward_quant outputs (oracle/gen_toy_golden.cpp, the
UNMODIFIED reference headers).  Run here, where the reference tree exists:

    make -C oracle ref && python tests/golden/make_toy_golden.py
"""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "tests", "golden", "toy", "toy.json")
os.makedirs(os.path.dirname(OUT), exist_ok=True)
text = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "gen_toy_golden")], check=True, capture_output=True,
                      text=True).stdout
json.loads(text)  # well-formed
with open(OUT, "w") as f:
    f.write(text)
print("wrote", OUT, len(text), "bytes")
