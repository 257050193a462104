"""First-light check on a B200: GPU assembly vs the reference library (oracle/_ref)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_07499_b200 as P
from oracle import ref

U = np.array([[1, 2, 0, 0], [1, 0, 2, 0], [1, 0, 0, 2]], float)

def dense_err(a, b, n):
    A = np.zeros((n, n)); B = np.zeros((n, n))
    for M, s in ((A, a), (B, b)):
        for i in range(n):
            M[i, s["col_idx"][s["row_ptr"][i]:s["row_ptr"][i+1]]] += s["values"][s["row_ptr"][i]:s["row_ptr"][i+1]]
    rowmax = np.abs(B).max(axis=1)
    return (np.abs(A - B).max(axis=1) / rowmax).max()

for res, delta, strat, mc in [(4, 0.3, "barycenter", 0), (4, 0.3, "nocaps", 0), (8, 0.25, "barycenter", 0),
                              (8, 0.25, "nocaps", 0), (8, 0.25, "fullcaps", 64)]:
    m = P.generate_mesh(3, res, delta)
    T = P.ElementTable(m["coords"], m["cells"], m["region"])
    t = time.time()
    try:
        S = P.Session(T, delta, strat, "moment2", U, seed=1234, mc_samples=max(mc, 1))
        st = S.run(); st = S.run()
        g = S.download()
    except Exception as e:
        print("GPU FAIL", res, strat, repr(e)); continue
    tg = time.time() - t
    R = ref.Problem(m["coords"], m["cells"], m["region"])
    r = R.assemble(delta, strat, U, threads=8, seed=1234, mc_samples=max(mc, 1))
    same_pat = np.array_equal(g["row_ptr"], r["row_ptr"]) and np.array_equal(g["col_idx"], r["col_idx"])
    msg = f"res={res} {strat}: nnz gpu {len(g['values'])} ref {len(r['values'])} pattern_equal={same_pat}"
    if same_pat:
        rm = np.zeros(len(r["rhs"]))
        for i in range(len(rm)):
            rm[i] = np.abs(r["values"][r["row_ptr"][i]:r["row_ptr"][i+1]]).max()
        rowidx = np.repeat(np.arange(len(rm)), np.diff(r["row_ptr"]))
        err = (np.abs(g["values"] - r["values"]) / rm[rowidx]).max()
        rerr = np.abs(g["rhs"] - r["rhs"]).max() / np.abs(r["rhs"]).max()
        msg += f" max_row_rel_err={err:.3e} rhs_rel={rerr:.3e}"
    l2g = R.solve_l2(g, U); l2r = R.solve_l2(r, U)
    msg += f" L2 gpu {l2g['l2']:.6e} ref {l2r['l2']:.6e}  dev_ms={st.device_ms:.2f} phases={[round(x,2) for x in st.phase_ms[:5]]} pairs={st.element_pairs} items={st.items} mc={st.mc_samples}/{st.mc_hits} ref_mc={r['mc_samples']}/{r['mc_hits']} ref_s={r['seconds']:.3f}"
    print(msg, flush=True)
