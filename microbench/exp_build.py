"""Build experiment variants of libiga (compile-time switches in kernels_gemm.cu) into
microbench/; load one with IGA_LIB=microbench/libiga_<name>.so.  Not part of the product."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_09568_b200 import build as B
HERE = os.path.dirname(os.path.abspath(__file__))
for name in sys.argv[1:]:   # NAME or NAME=VALUE; several joined by '+'
    defs = tuple(name.split("+"))
    tag = name.replace("=", "").replace("+", "_")
    print(B.build(force=True, defines=defs, lib=os.path.join(HERE, f"libiga_{tag}.so")))
