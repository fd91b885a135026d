"""One rank of a sharded solve over the CUDA IPC peer-store transport (tests/test_gpu_sharded.py).

    python tests/helpers/ipc_worker.py KIND N RANK WORLD DIR

Every rank runs on device 0 (one GPU, separate processes); the 512-byte export blobs are exchanged as files
in DIR.  Writes DIR/out_RANK.npz: the run report (iterations, trace) and the final iterate, plus x / r
(ISTA) or x / beta / v (cADMM) after the run."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1707_02244_b200 as cl  # noqa: E402
from paper_1707_02244_b200.dist import IpcPeers  # noqa: E402
from oracle import oracle as orc  # noqa: E402

kind, n, rank, world, d = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
p = orc.make_problem(n, n // 4, n // 256, 5)
op = cl.PartialCirculantOperator(cl.CirculantMatrix(p.row), cl.SubsamplingMask(p.omega, p.n))
cfg = cl.SolverConfig(max_iter=12, check_every=4, target_mse=1e-30)
st = (cl.ista_setup if kind == "ista" else cl.cadmm_setup)(op, p.y, cfg, device=0)


def exchange(blob):
    with open(os.path.join(d, f"blob_{rank}.tmp"), "wb") as f:
        f.write(blob)
    os.replace(os.path.join(d, f"blob_{rank}.tmp"), os.path.join(d, f"blob_{rank}"))
    t0 = time.time()
    while not all(os.path.exists(os.path.join(d, f"blob_{q}")) for q in range(world)):
        if time.time() - t0 > 120:
            raise TimeoutError("peer blobs did not arrive")
        time.sleep(0.05)
    return [open(os.path.join(d, f"blob_{q}"), "rb").read() for q in range(world)]


IpcPeers.connect(st, rank, world, exchange)
from paper_1707_02244_b200.api import _run  # noqa: E402
rep = _run(st, p.x_true, cfg)
fields = ("x", "r") if kind == "ista" else ("x", "beta", "v")
out = {f: st.get(f) for f in fields}
np.savez(os.path.join(d, f"out_{rank}.npz"), final_x=rep.final_x, iterations=rep.iterations,
         trace=np.array([(t.iteration, t.value) for t in rep.mse_trace]), **out)
del st  # collective: the final barrier
print(f"rank {rank}: {rep.iterations} iterations", flush=True)
