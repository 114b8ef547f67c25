"""Regenerate sass/*.sass from the built objects (selected instantiations, encodings stripped)."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2408_08554_b200", "csrc", "build")
WANT = {
    "gemv_dec": ["gemv_dec_kernelILi4ELi1ELi1E", "gemv_dec_kernelILi2ELi1ELi1E", "gemv_dec_kernelILi8ELi1ELi1E",
                 "gemv_dec_kernelILi4ELi1ELi0E"],
    "producer": ["rmsnorm_quant_kernel", "silu_mul_quant_kernel"],
    "gemm_tc": ["gemm_tc_kernelILi4ELi128E", "gemm_tc_kernelILi8ELi128E"],
    "gemv_popc": ["gemv_popc_kernelILi4ELi4ELi8ELi2ELb0ELb1E", "gemv_popc_kernelILi8ELi2ELi8ELi4ELb0ELb1E"],
    "gemv_imma": ["act_quant_kernelI6__halfLb0E", "act_quant_kernelI6__halfLb1E", "gemv_imma_kernelILi4ELi1ELb1E",
                  "prepack_frag_kernel"],
    "gemm_bmma": ["gemm_bmma_kernel"],
    "quant": ["bitpack_kernel", "quantize", "unpack", "rowsums"],
}
for f, keys in WANT.items():
    txt = subprocess.run(["cuobjdump", "-sass", os.path.join(BUILD, f + ".o")], capture_output=True, text=True).stdout
    out = []
    for fn in re.split(r"\n\s*Function : ", txt)[1:]:
        if any(k in fn.split("\n", 1)[0] for k in keys):
            lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", ln).rstrip() for ln in fn.split("\n")]
            out.append("Function : " + "\n".join(ln for ln in lines if ln.strip()))
    with open(os.path.join(ROOT, "sass", f + ".sass"), "w") as fh:
        fh.write(f"// cuobjdump -sass of paper_2408_08554_b200/csrc/build/{f}.o (sm_100a), selected instantiations, "
                 "encodings stripped\n" + "\n\n".join(out) + "\n")
    print(f, len(out))
