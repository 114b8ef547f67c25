"""Regenerate tests/golden/io/*.abq{t,p,z}: weight files written by the UNMODIFIED
reference's abq::io writers (oracle/gen_io_golden.cpp).  Run here, where the
reference tree exists:

    make -C oracle ref && python tests/golden/make_io_golden.py
"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "tests", "golden", "io")
os.makedirs(OUT, exist_ok=True)
subprocess.run([os.path.join(ROOT, "oracle", "_ref", "gen_io_golden"), OUT], check=True)
print("wrote", sorted(os.listdir(OUT)))
