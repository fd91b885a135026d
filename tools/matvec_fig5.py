"""The paper's Fig. 5 on one B200: circulant (direct engine) vs dense row-major matvec, n up to the
largest fp32 dense copy that fits (2^17: 64 GB).  Pinned bench CSV on stdout."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02244_b200 import io as cio

sizes = [int(a) for a in sys.argv[1:]] or [1 << k for k in range(10, 18)]
cio.matvec_bench(sizes, repeats=5, seed=1, dense_cap=1 << 17)
