"""TEST INFRASTRUCTURE ONLY -- a pure-Python restatement of the reference's
two-dimensional assemble (nlfem::assemble with et.n == 2, proj/src/assembly.cpp:
617-843) for small meshes, with the Monte Carlo caps drawn from the 2D Philox
stream of include/nlfem_mc_stream.h ("mode P"), so fullcaps can be compared
entry by entry with the GPU path (paper_2302_07499_b200 nlfem_gpu_assemble_2d).

Every geometric expression follows the reference operation by operation
(Python floats are IEEE doubles without FMA, like the reference's x86-64
build): classify_simplex (geometry.cpp:8-24), edge_sphere_crossing (26-37),
simplex_volume / barycentric / distance_point_simplex for n == 2 (59-71,
91-96, 129-139), straddle_inner / straddle_outer (ball_approx.cpp:232-240,
273-281), the AsmSink whole / sub / cap / flush (assembly.cpp:332-473) and
the per-(T, q, T') decision (722-760).  Entries are summed per key in FP64
(python dict, visit order); the reference's own sums differ in the last bits
only.  Mode R parity (barycenter / nocaps, no random numbers) is checked
against the unmodified reference in oracle/_ref instead.

Not imported by the product: only tests/ use it, as the checker."""
from __future__ import annotations

import math

import numpy as np

M32 = 0xFFFFFFFF
PHILOX_M0, PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
PHILOX_W0, PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
STRATS = ["inside", "overlap", "barycenter", "nocaps", "approxcaps", "fullcaps"]


def philox4x32_10(ctr, k0, k1):
    """Philox4x32-10 (include/nlfem_mc_stream.h nlfem_philox4x32_10)."""
    c0, c1, c2, c3 = ctr
    for _ in range(10):
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & M32, p1 & M32, ((p0 >> 32) ^ c3 ^ k1) & M32, \
            p0 & M32
        k0 = (k0 + PHILOX_W0) & M32
        k1 = (k1 + PHILOX_W1) & M32
    return c0, c1, c2, c3


def mc2_sample(W, c, v0, v1, v2):
    u0 = (float(W[2 * c]) + 0.5) * 2.0 ** -32
    u1 = (float(W[2 * c + 1]) + 0.5) * 2.0 ** -32
    if u0 > u1:
        u0, u1 = u1, u0
    l0, l1, l2 = u0, u1 - u0, 1.0 - u1
    return tuple((l0 * v0[a] + l1 * v1[a]) + l2 * v2[a] for a in range(3))


def sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def add(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def scale(s, a):
    return (s * a[0], s * a[1], s * a[2])


def dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def dist(a, b):
    return math.sqrt(dot(sub(a, b), sub(a, b)))


def area(a, b, c):
    x = cross(sub(b, a), sub(c, a))
    return 0.5 * math.sqrt(dot(x, x))


RB = [(0.5, 0.5, 0.0), (0.0, 0.5, 0.5), (0.5, 0.0, 0.5)]  # quadrature.cpp:17-21
W2 = 1.0 / 3.0


def qpoint(v, k):
    p = scale(RB[k][0], v[0])
    for i in (1, 2):
        p = add(p, scale(RB[k][i], v[i]))
    return p


def seg_dist(p, a, b):
    d = sub(b, a)
    len2 = dot(d, d)
    t = dot(sub(p, a), d) / len2 if len2 > 0 else 0.0
    t = min(max(t, 0.0), 1.0)
    return dist(p, add(a, scale(t, d)))


def dist_point_tri(p, v):
    e1, e2, b = sub(v[1], v[0]), sub(v[2], v[0]), sub(p, v[0])
    det = e1[0] * e2[1] - e1[1] * e2[0]
    l1 = (b[0] * e2[1] - b[1] * e2[0]) / det
    l2 = (e1[0] * b[1] - e1[1] * b[0]) / det
    l0 = 1.0 - l1 - l2
    if l0 >= 0 and l1 >= 0 and l2 >= 0:
        return 0.0
    d = seg_dist(p, v[0], v[1])
    d = min(d, seg_dist(p, v[1], v[2]))
    return min(d, seg_dist(p, v[2], v[0]))


def edge_crossing(a, b, c, r):
    d = sub(b, a)
    u = sub(a, c)
    A = dot(d, d)
    B = dot(u, d)
    Cc = dot(u, u) - r * r
    disc = B * B - A * Cc
    if disc < 0:
        disc = 0.0
    sq = math.sqrt(disc)
    t = (-B + sq) / A if B <= 0 else -Cc / (B + sq)
    return min(max(t, 0.0), 1.0)


def hull2d_pieces(pts, tau):
    """straddle_inner(sphere_points) for n == 2 (ball_approx.cpp:210-229):
    the reference's monotone-chain hull2d (geometry.cpp:161-196) and fan
    triangulation from the centroid of the hull vertices summed in index order
    (triangulate_polytope, geometry.cpp:307-329); pieces above tau."""
    idx = sorted(range(len(pts)), key=lambda i: (pts[i][0], pts[i][1]))
    uniq = []
    for i in idx:
        if uniq and pts[uniq[-1]][0] == pts[i][0] and pts[uniq[-1]][1] == pts[i][1]:
            continue
        uniq.append(i)

    def cr(o, a, b):
        return ((pts[a][0] - pts[o][0]) * (pts[b][1] - pts[o][1]) -
                (pts[a][1] - pts[o][1]) * (pts[b][0] - pts[o][0]))
    ring = []
    for i in uniq:
        while len(ring) >= 2 and cr(ring[-2], ring[-1], i) <= 0:
            ring.pop()
        ring.append(i)
    t = len(ring) + 1
    for i in reversed(uniq[:-1]):
        while len(ring) >= t and cr(ring[-2], ring[-1], i) <= 0:
            ring.pop()
        ring.append(i)
    if len(ring) < 4:
        return []  # DegenerateHull: caught by hull_pieces, no pieces
    ring = ring[:-1]
    facets = [(ring[i], ring[(i + 1) % len(ring)]) for i in range(len(ring))]
    vs = sorted(set(v for f in facets for v in f))
    c = (0.0, 0.0, 0.0)
    for v in vs:
        c = add(c, pts[v])
    c = scale(1.0 / float(len(vs)), c)
    out = []
    for f in facets:
        s = (c, pts[f[0]], pts[f[1]])
        if area(*s) > tau:
            out.append(s)
    return out


def poly_eval(terms, x):
    acc = 0.0
    for c, e0, e1, e2 in terms:
        v = float(c)
        for _ in range(int(e0)):
            v *= x[0]
        for _ in range(int(e1)):
            v *= x[1]
        for _ in range(int(e2)):
            v *= x[2]
        acc += v
    return acc


def assemble(t2, delta, strategy, C, f_terms, g_terms, seed=1234, mc_samples=16):
    """t2: paper_2302_07499_b200.ElementTable2D-like (node_xyz, verts, neighbor,
    center, radius, volume, diam, region, inv_edges, dof_of_node).  Returns the
    CSR dict plus mc_samples / mc_hits / element_pairs."""
    S = strategy
    node = [tuple(map(float, p)) for p in t2.node_xyz]
    K = len(t2.radius)
    V = [[node[int(t2.verts[t][i])] for i in range(3)] for t in range(K)]
    cen = [tuple(map(float, c)) for c in t2.center]
    rad = [float(r) for r in t2.radius]
    vol = [float(x) for x in t2.volume]
    tau = [1e-14 * math.pow(float(d), 2) for d in t2.diam]
    inv = [tuple(map(float, r)) for r in t2.inv_edges]
    dof = [int(d) for d in t2.dof_of_node]
    U = sum(1 for d in dof if d >= 0)
    gnode = [poly_eval(g_terms, node[v]) if dof[v] < 0 else 0.0 for v in range(len(node))]
    k0, k1 = seed & M32, (seed >> 32) & M32
    slack = 1e-10 * delta
    inside_cut = delta - slack - 1e-12 * delta
    r_in = delta - 1e-10 * delta
    rr = r_in * r_in
    mat, rhs = {}, {}
    draws = hits = 0
    pairs = set()

    def add_pair(da, na, db, nb, v):
        if da >= 0 and db >= 0:
            key = (min(da, db), max(da, db))
            mat[key] = mat.get(key, 0.0) + v
        elif da >= 0:
            rhs[da] = rhs.get(da, 0.0) - v * gnode[nb]
        elif db >= 0:
            rhs[db] = rhs.get(db, 0.0) - v * gnode[na]

    for T in range(K):
        if t2.region[T]:
            continue
        vT = V[T]
        nT = [int(t2.verts[T][a]) for a in range(3)]
        dT = [dof[n] for n in nT]
        for q in range(3):
            xq = qpoint(vT, q)
            w = W2 * vol[T]
            fv = poly_eval(f_terms, xq)
            for a in range(3):
                if dT[a] >= 0:
                    rhs[dT[a]] = rhs.get(dT[a], 0.0) + w * RB[q][a] * fv
            cN = RB[q]
            for tp in range(K):
                gap = dist(cen[tp], xq)
                if gap >= rad[tp] + delta:
                    continue
                vP = V[tp]
                cons = bool(t2.region[tp])
                acc = dict(S0=0.0, Sg=0.0, S1=[0.0] * 3, S2=[[0.0] * 3 for _ in range(3)], n=0)

                def acc_point(y, wt):
                    acc["S0"] += wt
                    if cons:
                        acc["Sg"] += wt * poly_eval(g_terms, y)
                        return
                    d = sub(y, vP[0])
                    iv = inv[tp]
                    b1 = iv[0] * d[0] + iv[1] * d[1]
                    b2 = iv[2] * d[0] + iv[3] * d[1]
                    b = (1.0 - b1 - b2, b1, b2)
                    for i in range(3):
                        wb = wt * b[i]
                        acc["S1"][i] += wb
                        for j in range(3):
                            acc["S2"][i][j] += wb * b[j]

                def whole():
                    acc["n"] += 1
                    v = vol[tp]
                    acc["S0"] += v
                    if cons:
                        for k in range(3):
                            acc["Sg"] += v * W2 * poly_eval(g_terms, qpoint(vP, k))
                        return
                    s1, off = v / 3.0, v / float(3 * 4)
                    for i in range(3):
                        acc["S1"][i] += s1
                        for j in range(3):
                            acc["S2"][i][j] += off * (2.0 if i == j else 1.0)

                def subp(s):
                    acc["n"] += 1
                    v = area(*s)
                    for k in range(3):
                        acc_point(qpoint(s, k), v * W2)

                def cap(pieces):
                    nonlocal draws, hits
                    acc["n"] += 1
                    for si, s in enumerate(pieces):
                        wt = area(*s) / mc_samples
                        W = None
                        for k in range(mc_samples):
                            if k % 2 == 0:
                                W = philox4x32_10((T, tp, q | (si << 2), k >> 1), k0, k1)
                            y = mc2_sample(W, k % 2, *s)
                            draws += 1
                            d = sub(y, xq)
                            if dot(d, d) >= delta * delta:
                                continue
                            hits += 1
                            acc_point(y, wt)

                if S == "barycenter":
                    if gap < delta:
                        whole()
                elif S == "overlap":
                    if gap + rad[tp] < delta or dist_point_tri(xq, vP) < delta:
                        whole()
                else:
                    if gap + rad[tp] < inside_cut:
                        whole()
                    else:
                        ins = [i for i in range(3) if dot(sub(vP[i], xq), sub(vP[i], xq)) < rr]
                        outs = [i for i in range(3) if i not in ins]
                        if len(ins) == 3:
                            whole()
                        elif ins:
                            if S == "inside":
                                continue
                            X = []
                            for i in ins:
                                for o in outs:
                                    tt = edge_crossing(vP[i], vP[o], xq, delta)
                                    X.append(add(vP[i], scale(tt, sub(vP[o], vP[i]))))
                            if S == "approxcaps":
                                pts = [vP[i] for i in ins] + X
                                cr_i = [(i, o) for i in ins for o in outs]
                                for a in range(len(X)):
                                    for b in range(a + 1, len(X)):
                                        if cr_i[a][0] != cr_i[b][0] and cr_i[a][1] != cr_i[b][1]:
                                            continue
                                        mid = sub(scale(0.5, add(X[a], X[b])), xq)
                                        ln = math.sqrt(dot(mid, mid))
                                        if ln <= 0:
                                            continue
                                        pts.append(add(xq, scale(delta / ln, mid)))
                                for s in hull2d_pieces(pts, tau[tp]):
                                    subp(s)
                            else:
                                if len(ins) == 1:
                                    inner = [(vP[ins[0]], X[0], X[1])]
                                else:
                                    inner = [(vP[ins[0]], vP[ins[1]], X[1]),
                                             (vP[ins[0]], X[1], X[0])]
                                for s in inner:
                                    if area(*s) > tau[tp]:
                                        subp(s)
                            if S == "fullcaps":
                                if len(ins) == 1:
                                    outer = [(vP[outs[0]], vP[outs[1]], X[1]),
                                             (vP[outs[0]], X[1], X[0])]
                                else:
                                    outer = [(vP[outs[0]], X[0], X[1])]
                                kept = [s for s in outer if area(*s) > tau[tp]]
                                if kept:
                                    cap(kept)
                        elif S == "fullcaps" and dist_point_tri(xq, vP) < delta:
                            cap([tuple(vP)])
                if acc["n"] == 0:
                    continue
                pairs.add((T, tp))
                # flush (assembly.cpp:413-473)
                if cons:
                    base = w * 2.0 * C
                    for a in range(3):
                        if dT[a] >= 0:
                            rhs[dT[a]] = rhs.get(dT[a], 0.0) + base * acc["Sg"] * cN[a]
                        for b in range(a, 3):
                            add_pair(dT[a], nT[a], dT[b], nT[b], base * acc["S0"] * cN[a] * cN[b])
                    continue
                vm = [int(t2.verts[tp][j]) for j in range(3)]
                Ul = []
                for a in range(3):
                    ms = vm.index(nT[a]) if nT[a] in vm else -1
                    Ul.append((nT[a], dT[a], cN[a], ms))
                for j in range(3):
                    if vm[j] not in nT:
                        Ul.append((vm[j], dof[vm[j]], 0.0, j))
                sc = C * w
                for x in range(len(Ul)):
                    s1x = acc["S1"][Ul[x][3]] if Ul[x][3] >= 0 else 0.0
                    for y in range(x, len(Ul)):
                        s1y = acc["S1"][Ul[y][3]] if Ul[y][3] >= 0 else 0.0
                        s2 = (acc["S2"][Ul[x][3]][Ul[y][3]] if Ul[x][3] >= 0 and Ul[y][3] >= 0
                              else 0.0)
                        v = sc * (s2 - Ul[x][2] * s1y - Ul[y][2] * s1x + Ul[x][2] * Ul[y][2] *
                                  acc["S0"])
                        add_pair(Ul[x][1], Ul[x][0], Ul[y][1], Ul[y][0], v)
    # CSR expansion (assembly.cpp:789-833)
    rows = [[] for _ in range(U)]
    for (a, b), v in mat.items():
        rows[a].append((b, v))
        if a != b:
            rows[b].append((a, v))
    rp, ci, va = [0], [], []
    for r in rows:
        r.sort()
        ci += [c for c, _ in r]
        va += [v for _, v in r]
        rp.append(len(ci))
    return {"row_ptr": np.array(rp, np.int32), "col_idx": np.array(ci, np.int32),
            "values": np.array(va), "rhs": np.array([rhs.get(i, 0.0) for i in range(U)]),
            "mc_samples": draws, "mc_hits": hits, "element_pairs": len(pairs)}
