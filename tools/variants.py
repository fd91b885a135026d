"""Kernel-variant sweep (experiment driver, not the bench).

    python tools/variants.py GRAD:RES [GRAD:RES ...]     e.g. 1:1 2:1 1:2   (table indices, csrc/kernels.cu)

Each pair runs in its own process (CLB_GRAD / CLB_RES select a variant of the
sparse kernels at library load).  Per variant: C3 ISTA, per-phase kernel times
(CUDA events, L2 not flushed, mean of 3 iterations), and r / delta after one
iteration compared with the first pair's (rel l2; different tilings only
change the fp32 summation grouping).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(n, m, k, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_1707_02244_b200 as cl
    p = cl.make_problem(n, m, k, 1)
    st = cl.ista_setup(p.op, p.measurements)
    st.step(1)
    st.synchronize()
    r, d = st.get("r"), st.get("delta")
    np.save(out + "_r.npy", r)
    np.save(out + "_d.npy", d)
    st.profile(True)
    ph = []
    for _ in range(3):
        st.step(1)
        st.synchronize()
        ph.append(st.phase_ms())
    print(json.dumps({"phase_ms": [sum(p[i] for p in ph) / len(ph) for i in range(len(ph[0]))]}))


def main():
    if sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
        return
    import numpy as np
    n, m, k = 1 << 20, 1 << 18, 1 << 12
    pairs = sys.argv[1:]
    if pairs and pairs[0].startswith("n="):
        n = int(pairs[0][2:]); m = n // 4; k = max(1, n // 256); pairs = pairs[1:]
    base = None
    for pr in pairs:
        g, r = pr.split(":")
        env = dict(os.environ, CLB_GRAD=g, CLB_RES=r)
        out = f"/tmp/var_{g}_{r}"
        res = subprocess.run([sys.executable, __file__, "--child", str(n), str(m), str(k), out], env=env,
                             capture_output=True, text=True, timeout=600)
        if res.returncode != 0:
            print(pr, "FAILED", res.stderr[-2000:], flush=True)
            continue
        ph = json.loads(res.stdout.strip().splitlines()[-1])["phase_ms"]
        rr, dd = np.load(out + "_r.npy"), np.load(out + "_d.npy")
        if base is None:
            base = (rr, dd)
        er = np.linalg.norm(rr - base[0]) / np.linalg.norm(base[0])
        ed = np.linalg.norm(dd - base[1]) / np.linalg.norm(base[1])
        print(f"grad {g:>2} res {r:>2}: residual {ph[0]:8.3f} ms  gradient {ph[2]:8.3f} ms  "
              f"step {sum(ph):8.3f} ms   rel(r) {er:.2e} rel(delta) {ed:.2e}", flush=True)


if __name__ == "__main__":
    main()
