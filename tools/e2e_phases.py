"""Wall-clock phases of solve_decomposed on config 4, five solves in one process
(session create, loop, classify/report, close)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_01828_b200 as H  # noqa: E402
from paper_1611_01828_b200 import solver as S  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

cp = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
H.solve_decomposed(make_config(0), H.SolverSettings())
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    cp._cache.pop("pattern_index", None)
    st = H.SolverSettings()
    t0 = time.perf_counter()
    sess = S._Session(cp, st, st.normalize)
    t1 = time.perf_counter()
    k, chk = 0, None
    while k < st.max_iters:
        sess.h.iterate(20)
        k += 20
        chk = sess.h.check()
        if max(float(chk[0]), float(chk[1]), float(chk[2])) <= st.tol:
            break
    t2 = time.perf_counter()
    rep_ = S._classify(sess, chk, k, S.Timing(setup_s=t1 - t0, iterations_s=t2 - t1, total_s=t2 - t0,
                                               per_iteration_s=(t2 - t1) / k))
    t3 = time.perf_counter()
    sess.h.close()
    t4 = time.perf_counter()
    print(f"solve {rep}: session {1e3 * (t1 - t0):.1f} ms, loop {1e3 * (t2 - t1):.1f} ms ({k} it), "
          f"classify {1e3 * (t3 - t2):.1f} ms, close {1e3 * (t4 - t3):.1f} ms, total {1e3 * (t4 - t0):.1f} ms; {rep_.status}",
          flush=True)
os.environ["HSDE_TIMING"] = "1"
sess = S._Session(cp, st, st.normalize)
sess.h.close()
