"""Dense-kernel variant sweep (cADMM n=2^20 products): python tools/dense_variants.py 0 1 2 ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_1707_02244_b200 as cl
    n = 1 << 20
    p = cl.make_problem(n, n // 4, n // 256, 1)
    st = cl.cadmm_setup(p.op, p.measurements)
    st.step(2); st.synchronize()
    np.save(sys.argv[2], st.get("z"))
    st.profile(True); st.step(1); st.synchronize()
    print(json.dumps(st.phase_ms()))
    sys.exit(0)
import numpy as np
base = None
for v in sys.argv[1:]:
    out = f"/tmp/dense_{v}.npy"
    r = subprocess.run([sys.executable, __file__, "--child", out], env=dict(os.environ, CLB_DENSE=v),
                       capture_output=True, text=True)
    if r.returncode:
        print(v, "FAILED", r.stderr[-1500:]); continue
    ph = json.loads(r.stdout.strip().splitlines()[-1])
    z = np.load(out)
    base = z if base is None else base
    print(f"dense {v}: products {ph[0]:.2f} / {ph[2]:.2f} / {ph[4]:.2f} ms  rel(z) {np.linalg.norm(z-base)/np.linalg.norm(base):.2e}", flush=True)
