"""femopt kernel-IR generator for the five BASELINE forms.

The reference's hot path is the element kernel femopt emits from a loop-nest
IR (/root/reference/proj/src/emit_c.cpp:108-174); its input format is the
JSON documented at proj/README.md:68-100 and parsed by
proj/src/json_io.cpp:156-221 (strict: unknown keys rejected, subscripts are
loop indices only, tables row-major over named dims).  This module writes that
IR for our forms so the reference can optimize, interpret and emit them; it
also fixes the naming convention the C ABI's ``femgpu_kernel_argv`` follows
(argument order = emitted-C order: outputs, input tables, constants, each
sorted by name, emit_c.cpp:137-140).

Per-cell data are e-indexed SoA tables, one per scalar: vertex coordinates
``x{v}{c}[e]`` and coefficient dofs (``f{mm}``, ``mu{m}``, ``lam{m}``,
``w{c}{mm}``, ``u{c}{mm}``), because IR subscripts must be loop indices
(SURVEY.md §8a a0).  The element matrix is ``A[e][j][k]`` (or one
``A{c}{d}[e][j][k]`` block per kernel for Burgers, whose monolithic IR exceeds
femopt's exact-cover limit, sharing.cpp:355).

Two encodings:
  * ``ufl``  -- quadrature style: (sum_a K_ab D_a[i,j]) (sum_a K_ab D_a[i,k]),
  * ``gfac`` -- geometry-factored: sum_ab G_ab[e] D_a[i,j] D_b[i,k]
                (Helmholtz only).
"""
from __future__ import annotations

import json

import numpy as np

from . import fe

# ----------------------------------------------------------------------------
# S-expression helpers (proj/README.md:96-100)
# ----------------------------------------------------------------------------


def S(name, *idx):
    return ["sym", name, *idx] if idx else name


def add(*terms):
    terms = [t for t in terms if t is not None]
    return terms[0] if len(terms) == 1 else ["+", *terms]


def mul(*factors):
    return factors[0] if len(factors) == 1 else ["*", *factors]


def sub(a, b):
    return add(a, mul(-1.0, b))


def stmt(level, lhs, rhs, op="="):
    return {"level": level, "lhs": lhs, "op": op, "rhs": rhs}


def table(dims, values):
    return {"dims": list(dims), "values": [float(v) for v in np.asarray(values).reshape(-1)]}


# ----------------------------------------------------------------------------
# Shared pieces
# ----------------------------------------------------------------------------


def geometry_statements():
    """Level-1 affine geometry: J, cofactors, det, K = J^-1, |det J|.

    J_ab = dx_a/dX_b = x_{b+1,a} - x_{0,a};  K_ab = dX_a/dx_b = cof(J)_ba/det.
    """
    st = []
    for a in range(3):
        for b in range(3):
            st.append(stmt(1, f"J{a}{b}", sub(S(f"x{b+1}{a}", "e"), S(f"x0{a}", "e"))))

    def J(a, b):
        return f"J{a}{b}"

    cof = {}
    for a in range(3):
        for b in range(3):
            a1, a2 = [r for r in range(3) if r != a]
            b1, b2 = [c for c in range(3) if c != b]
            sign = 1.0 if (a + b) % 2 == 0 else -1.0
            t = sub(mul(J(a1, b1), J(a2, b2)), mul(J(a1, b2), J(a2, b1)))
            cof[a, b] = t if sign > 0 else sub(mul(J(a1, b2), J(a2, b1)), mul(J(a1, b1), J(a2, b2)))
            st.append(stmt(1, f"C{a}{b}", cof[a, b]))
    st.append(stmt(1, "det", add(mul(J(0, 0), "C00"), mul(J(0, 1), "C01"), mul(J(0, 2), "C02"))))
    st.append(stmt(1, "rdet", ["/", 1.0, "det"]))
    st.append(stmt(1, "adet", ["call", "fabs", "det"]))
    for a in range(3):
        for b in range(3):
            st.append(stmt(1, f"K{a}{b}", mul(f"C{b}{a}", "rdet")))
    return st


def geometry_tables(coords):
    """x{v}{c}[e] SoA tables from cell-major coords [E][4][3]."""
    return {f"x{v}{c}": table(["e"], coords[:, v, c]) for v in range(4) for c in range(3)}


def coef_sum(names, ptabs):
    """sum_m name_m[e] * P_m[i] -- an interpolated coefficient at a point."""
    return add(*[mul(S(n, "e"), S(p, "i")) for n, p in zip(names, ptabs)])


def grad(Dname, jk, beta):
    """Physical derivative d/dx_beta of basis ``jk``: sum_a K_a,beta D_a[i,jk]."""
    return add(*[mul(f"K{a}{beta}", S(Dname(a), "i", jk)) for a in range(3)])


def base(cfg, E, Q, n):
    return {
        "indices": {"e": E, "i": Q, "j": n, "k": n},
        "loops": [{"index": "e", "class": "orderfree"}, {"index": "i"}, {"index": "j"},
                  {"index": "k"}],
        "tables": {},
        "constants": {},
        "statements": geometry_statements(),
        "outputs": ["A"],
    }


# ----------------------------------------------------------------------------
# Forms
# ----------------------------------------------------------------------------


def helmholtz(cfg, coords, coeffs, tabs, encoding="ufl"):
    E, Q, n = coords.shape[0], tabs.W.shape[0], cfg.ns
    nc = tabs.P.shape[1]
    k = base(cfg, E, Q, n)
    T = k["tables"]
    T.update(geometry_tables(coords))
    T["W"] = table(["i"], tabs.W)
    T["B"] = table(["i", "j"], tabs.B)
    for a in range(3):
        T[f"D{a}"] = table(["i", "j"], tabs.D[a])
    fn = [f"f{m:02d}" for m in range(nc)]
    pn = [f"P{m:02d}" for m in range(nc)]
    for m in range(nc):
        T[fn[m]] = table(["e"], coeffs[:, m])
        T[pn[m]] = table(["i"], tabs.P[:, m])
    fq = coef_sum(fn, pn)
    D = lambda a: f"D{a}"  # noqa: E731
    mass = mul(S("B", "i", "j"), S("B", "i", "k"))
    if encoding == "ufl":
        stiff = add(*[mul(grad(D, "j", b), grad(D, "k", b)) for b in range(3)])
        rhs = mul(add(stiff, mass), fq, S("W", "i"), "adet")
    elif encoding == "gfac":
        for a in range(3):
            for b in range(3):
                k["statements"].append(stmt(1, f"G{a}{b}", mul(
                    add(*[mul(f"K{a}{g}", f"K{b}{g}") for g in range(3)]), "adet")))
        monos = [mul(f"G{a}{b}", S(f"D{a}", "i", "j"), S(f"D{b}", "i", "k"), fq, S("W", "i"))
                 for a in range(3) for b in range(3)]
        monos.append(mul("adet", S("B", "i", "j"), S("B", "i", "k"), fq, S("W", "i")))
        rhs = add(*monos)
    else:
        raise ValueError(encoding)
    k["statements"].append(stmt(4, ["A", "e", "j", "k"], rhs, "+="))
    return k


def _padded(tabs, ns):
    """Component-padded vector tables Dv{c}{a}[i][c'*ns+j] (FFC padding rule)."""
    Q = tabs.W.shape[0]
    out = {}
    for c in range(3):
        for a in range(3):
            v = np.zeros((Q, 3 * ns))
            v[:, c * ns:(c + 1) * ns] = tabs.D[a]
            out[f"Dv{c}{a}"] = v
    return out


def elasticity(cfg, coords, coeffs, tabs, encoding="ufl"):
    E, Q, ns = coords.shape[0], tabs.W.shape[0], cfg.ns
    k = base(cfg, E, Q, 3 * ns)
    T = k["tables"]
    T.update(geometry_tables(coords))
    T["W"] = table(["i"], tabs.W)
    for name, v in _padded(tabs, ns).items():
        T[name] = table(["i", "j"], v)
    for m in range(4):
        T[f"P{m}"] = table(["i"], tabs.P[:, m])
        T[f"mu{m}"] = table(["e"], coeffs[:, m])
        T[f"lam{m}"] = table(["e"], coeffs[:, 4 + m])
    muq = coef_sum([f"mu{m}" for m in range(4)], [f"P{m}" for m in range(4)])
    lamq = coef_sum([f"lam{m}" for m in range(4)], [f"P{m}" for m in range(4)])

    def g(jk, c, b):
        return grad(lambda a: f"Dv{c}{a}", jk, b)

    def eps(jk, c, b):
        return mul(0.5, add(g(jk, c, b), g(jk, b, c)))

    epseps = add(*[mul(eps("j", c, b), eps("k", c, b)) for c in range(3) for b in range(3)])
    divdiv = mul(add(*[g("j", c, c) for c in range(3)]), add(*[g("k", c, c) for c in range(3)]))
    rhs = mul(add(mul(2.0, muq, epseps), mul(lamq, divdiv)), S("W", "i"), "adet")
    k["statements"].append(stmt(4, ["A", "e", "j", "k"], rhs, "+="))
    return k


def hyperelasticity(cfg, coords, coeffs, tabs, encoding="ufl"):
    """St Venant--Kirchhoff tangent a(du,v) = int (grad du S + F dS[du]) : grad v.

    F = I + grad w, E = (F^T F - I)/2, S = lam tr(E) I + 2 mu E,
    dS = lam tr(dE) I + 2 mu dE, dE = sym(F^T grad du).  Body force and
    traction are linear in v and independent of u, so they do not enter the
    Jacobian ("Hyperelasticity form").
    """
    E, Q, ns = coords.shape[0], tabs.W.shape[0], cfg.ns
    k = base(cfg, E, Q, 3 * ns)
    T = k["tables"]
    T.update(geometry_tables(coords))
    T["W"] = table(["i"], tabs.W)
    for name, v in _padded(tabs, ns).items():
        T[name] = table(["i", "j"], v)
    for m in range(4):
        T[f"P{m}"] = table(["i"], tabs.P[:, m])
        T[f"mu{m}"] = table(["e"], coeffs[:, 3 * ns + m])
        T[f"lam{m}"] = table(["e"], coeffs[:, 3 * ns + 4 + m])
    for a in range(3):
        for m in range(ns):
            T[f"Dw{a}{m:02d}"] = table(["i"], tabs.D[a][:, m])
    for c in range(3):
        for m in range(ns):
            T[f"w{c}{m:02d}"] = table(["e"], coeffs[:, c * ns + m])
    st = k["statements"]
    st.append(stmt(2, "muq", coef_sum([f"mu{m}" for m in range(4)], [f"P{m}" for m in range(4)])))
    st.append(stmt(2, "lamq", coef_sum([f"lam{m}" for m in range(4)], [f"P{m}" for m in range(4)])))
    for c in range(3):
        for b in range(3):
            gw = add(*[mul(S(f"w{c}{m:02d}", "e"),
                           add(*[mul(f"K{a}{b}", S(f"Dw{a}{m:02d}", "i")) for a in range(3)]))
                       for m in range(ns)])
            st.append(stmt(2, f"F{c}{b}", add(1.0, gw) if c == b else gw))
    for a in range(3):
        for b in range(3):
            ftf = add(*[mul(f"F{p}{a}", f"F{p}{b}") for p in range(3)])
            st.append(stmt(2, f"E{a}{b}", mul(0.5, add(ftf, -1.0) if a == b else ftf)))
    st.append(stmt(2, "trE", add("E00", "E11", "E22")))
    for a in range(3):
        for b in range(3):
            s2 = mul(2.0, "muq", f"E{a}{b}")
            st.append(stmt(2, f"S{a}{b}", add(mul("lamq", "trE"), s2) if a == b else s2))

    def g(jk, c, b):
        return grad(lambda a: f"Dv{c}{a}", jk, b)

    trdE = add(*[mul(f"F{p}{q}", g("k", p, q)) for p in range(3) for q in range(3)])
    terms = []
    for c in range(3):
        for b in range(3):
            geo = add(*[mul(g("k", c, q), f"S{q}{b}") for q in range(3)])
            mat1 = mul("lamq", trdE, f"F{c}{b}")
            mat2 = mul("muq", add(*[mul(f"F{c}{q}", add(*[add(mul(g("k", p, q), f"F{p}{b}"),
                                                              mul(f"F{p}{q}", g("k", p, b)))
                                                          for p in range(3)]))
                                    for q in range(3)]))
            terms.append(mul(g("j", c, b), add(geo, mat1, mat2)))
    rhs = mul(add(*terms), S("W", "i"), "adet")
    st.append(stmt(4, ["A", "e", "j", "k"], rhs, "+="))
    return k


def burgers_block(cfg, coords, coeffs, tabs, c, d, encoding="ufl"):
    """Block (c,d) of the Burgers Jacobian as its own kernel.

    A_{cj,dk} = int phi_j phi_k (du_c/dx_d + delta_cd/dt)
                    + delta_cd (phi_j (u . grad phi_k) + nu grad phi_j . grad phi_k).
    """
    E, Q, ns = coords.shape[0], tabs.W.shape[0], cfg.ns
    k = base(cfg, E, Q, ns)
    name = f"A{c}{d}"
    k["outputs"] = [name]
    T = k["tables"]
    T.update(geometry_tables(coords))
    T["W"] = table(["i"], tabs.W)
    T["B"] = table(["i", "j"], tabs.B)
    for a in range(3):
        T[f"D{a}"] = table(["i", "j"], tabs.D[a])
    for m in range(ns):
        T[f"P{m:02d}"] = table(["i"], tabs.B[:, m])
        for a in range(3):
            T[f"Du{a}{m:02d}"] = table(["i"], tabs.D[a][:, m])
        for cc in range(3):
            T[f"u{cc}{m:02d}"] = table(["e"], coeffs[:, cc * ns + m])
    nu, dt = cfg.consts
    k["constants"] = {"nu": nu, "dt": dt}
    k["statements"].append(stmt(1, "rdt", ["/", 1.0, "dt"]))
    D = lambda a: f"D{a}"  # noqa: E731
    gu = add(*[mul(S(f"u{c}{m:02d}", "e"), add(*[mul(f"K{a}{d}", S(f"Du{a}{m:02d}", "i"))
                                                for a in range(3)])) for m in range(ns)])
    mass = mul(S("B", "i", "j"), S("B", "i", "k"))
    if c == d:
        uq = [coef_sum([f"u{mm}{m:02d}" for m in range(ns)], [f"P{m:02d}" for m in range(ns)])
              for mm in range(3)]
        adv = mul(S("B", "i", "j"), add(*[mul(uq[b], grad(D, "k", b)) for b in range(3)]))
        diff = mul("nu", add(*[mul(grad(D, "j", b), grad(D, "k", b)) for b in range(3)]))
        rhs = mul(add(mul(mass, add(gu, "rdt")), adv, diff), S("W", "i"), "adet")
    else:
        rhs = mul(mass, gu, S("W", "i"), "adet")
    k["statements"].append(stmt(4, [name, "e", "j", "k"], rhs, "+="))
    return k


# ----------------------------------------------------------------------------
# Arity-1 kernels: element vectors (femopt validates
# linear nests of arity 1, kernel.cpp:369-390)
# ----------------------------------------------------------------------------


def base_vector(E, Q, n, out="b"):
    return {
        "indices": {"e": E, "i": Q, "j": n},
        "loops": [{"index": "e", "class": "orderfree"}, {"index": "i"}, {"index": "j"}],
        "tables": {},
        "constants": {},
        "statements": geometry_statements(),
        "outputs": [out],
    }


def helmholtz_load(cfg, coords, coeffs, tabs):
    """Load vector of the Helmholtz configs: b_j = int f phi_j."""
    E, Q, n = coords.shape[0], tabs.W.shape[0], cfg.ns
    nc = tabs.P.shape[1]
    k = base_vector(E, Q, n, "b")
    T = k["tables"]
    T.update(geometry_tables(coords))
    T["W"] = table(["i"], tabs.W)
    T["B"] = table(["i", "j"], tabs.B)
    fn = [f"f{m:02d}" for m in range(nc)]
    pn = [f"P{m:02d}" for m in range(nc)]
    for m in range(nc):
        T[fn[m]] = table(["e"], coeffs[:, m])
        T[pn[m]] = table(["i"], tabs.P[:, m])
    rhs = mul(coef_sum(fn, pn), S("B", "i", "j"), S("W", "i"), "adet")
    k["statements"].append(stmt(3, ["b", "e", "j"], rhs, "+="))
    return k


def hyperelasticity_residual(cfg, coords, coeffs, tabs):
    """St Venant--Kirchhoff internal virtual work r_(c,j) = int (F S) : grad(phi_j e_c),
    the residual whose Jacobian is ``hyperelasticity`` (F, E, S as there)."""
    E, Q, ns = coords.shape[0], tabs.W.shape[0], cfg.ns
    k = base_vector(E, Q, 3 * ns, "r")
    T = k["tables"]
    T.update(geometry_tables(coords))
    T["W"] = table(["i"], tabs.W)
    for name, v in _padded(tabs, ns).items():
        T[name] = table(["i", "j"], v)
    for m in range(4):
        T[f"P{m}"] = table(["i"], tabs.P[:, m])
        T[f"mu{m}"] = table(["e"], coeffs[:, 3 * ns + m])
        T[f"lam{m}"] = table(["e"], coeffs[:, 3 * ns + 4 + m])
    for a in range(3):
        for m in range(ns):
            T[f"Dw{a}{m:02d}"] = table(["i"], tabs.D[a][:, m])
    for c in range(3):
        for m in range(ns):
            T[f"w{c}{m:02d}"] = table(["e"], coeffs[:, c * ns + m])
    st = k["statements"]
    st.append(stmt(2, "muq", coef_sum([f"mu{m}" for m in range(4)], [f"P{m}" for m in range(4)])))
    st.append(stmt(2, "lamq", coef_sum([f"lam{m}" for m in range(4)], [f"P{m}" for m in range(4)])))
    for c in range(3):
        for b in range(3):
            gw = add(*[mul(S(f"w{c}{m:02d}", "e"),
                           add(*[mul(f"K{a}{b}", S(f"Dw{a}{m:02d}", "i")) for a in range(3)]))
                       for m in range(ns)])
            st.append(stmt(2, f"F{c}{b}", add(1.0, gw) if c == b else gw))
    for a in range(3):
        for b in range(3):
            ftf = add(*[mul(f"F{p}{a}", f"F{p}{b}") for p in range(3)])
            st.append(stmt(2, f"E{a}{b}", mul(0.5, add(ftf, -1.0) if a == b else ftf)))
    st.append(stmt(2, "trE", add("E00", "E11", "E22")))
    for a in range(3):
        for b in range(3):
            s2 = mul(2.0, "muq", f"E{a}{b}")
            st.append(stmt(2, f"S{a}{b}", add(mul("lamq", "trE"), s2) if a == b else s2))
    for c in range(3):
        for b in range(3):
            st.append(stmt(2, f"Pk{c}{b}", add(*[mul(f"F{c}{q}", f"S{q}{b}") for q in range(3)])))

    def g(c, b):
        return grad(lambda a: f"Dv{c}{a}", "j", b)

    rhs = mul(add(*[mul(f"Pk{c}{b}", g(c, b)) for c in range(3) for b in range(3)]),
              S("W", "i"), "adet")
    st.append(stmt(3, ["r", "e", "j"], rhs, "+="))
    return k


def burgers_residual(cfg, coords, coeffs, tabs):
    """Burgers residual r_(c,j) = int (u_c/dt + (u.grad) u_c) phi_j + nu grad u_c . grad phi_j,
    whose Jacobian is the ``burgers_block`` kernels."""
    E, Q, ns = coords.shape[0], tabs.W.shape[0], cfg.ns
    k = base_vector(E, Q, 3 * ns, "r")
    T = k["tables"]
    T.update(geometry_tables(coords))
    T["W"] = table(["i"], tabs.W)
    for c in range(3):
        v = np.zeros((Q, 3 * ns))
        v[:, c * ns:(c + 1) * ns] = tabs.B
        T[f"Bv{c}"] = table(["i", "j"], v)
    for name, v in _padded(tabs, ns).items():
        T[name] = table(["i", "j"], v)
    for m in range(ns):
        T[f"P{m:02d}"] = table(["i"], tabs.B[:, m])
        for a in range(3):
            T[f"Du{a}{m:02d}"] = table(["i"], tabs.D[a][:, m])
        for cc in range(3):
            T[f"u{cc}{m:02d}"] = table(["e"], coeffs[:, cc * ns + m])
    nu, dt = cfg.consts
    k["constants"] = {"nu": nu, "dt": dt}
    st = k["statements"]
    st.append(stmt(1, "rdt", ["/", 1.0, "dt"]))
    for c in range(3):
        st.append(stmt(2, f"uq{c}", coef_sum([f"u{c}{m:02d}" for m in range(ns)],
                                             [f"P{m:02d}" for m in range(ns)])))
        for b in range(3):
            st.append(stmt(2, f"gu{c}{b}", add(*[
                mul(S(f"u{c}{m:02d}", "e"), add(*[mul(f"K{a}{b}", S(f"Du{a}{m:02d}", "i"))
                                                 for a in range(3)])) for m in range(ns)])))
    for c in range(3):
        st.append(stmt(2, f"adv{c}", add(mul(f"uq{c}", "rdt"),
                                         *[mul(f"uq{b}", f"gu{c}{b}") for b in range(3)])))

    def g(c, b):
        return grad(lambda a: f"Dv{c}{a}", "j", b)

    terms = []
    for c in range(3):
        terms.append(mul(f"adv{c}", S(f"Bv{c}", "i", "j")))
        terms.append(mul("nu", add(*[mul(f"gu{c}{b}", g(c, b)) for b in range(3)])))
    rhs = mul(add(*terms), S("W", "i"), "adet")
    st.append(stmt(3, ["r", "e", "j"], rhs, "+="))
    return k


VECTOR_FORMS = {
    fe.HELMHOLTZ: ("b", helmholtz_load),
    fe.HYPERELASTICITY: ("r", hyperelasticity_residual),
    fe.BURGERS: ("r", burgers_residual),
}


def build_vector(cfg, coords, coeffs, tabs=None):
    """Arity-1 kernel of a config's form family: (output_name, ir_dict)."""
    tabs = tabs if tabs is not None else fe.tables(cfg)
    if cfg.kind not in VECTOR_FORMS:
        raise ValueError(f"no element-vector form for kind {cfg.kind}")
    name, fn = VECTOR_FORMS[cfg.kind]
    return name, fn(cfg, np.asarray(coords, dtype=np.float64),
                    np.asarray(coeffs, dtype=np.float64), tabs)


def build(cfg, coords, coeffs, tabs=None, encoding="ufl"):
    """IR kernel(s) for a config: a list of (output_name, ir_dict)."""
    tabs = tabs if tabs is not None else fe.tables(cfg)
    coords = np.asarray(coords, dtype=np.float64)
    coeffs = np.asarray(coeffs, dtype=np.float64)
    if cfg.kind == fe.HELMHOLTZ:
        return [("A", helmholtz(cfg, coords, coeffs, tabs, encoding))]
    if cfg.kind == fe.ELASTICITY:
        return [("A", elasticity(cfg, coords, coeffs, tabs, encoding))]
    if cfg.kind == fe.HYPERELASTICITY:
        return [("A", hyperelasticity(cfg, coords, coeffs, tabs, encoding))]
    if cfg.kind == fe.BURGERS:
        return [(f"A{c}{d}", burgers_block(cfg, coords, coeffs, tabs, c, d, encoding))
                for c in range(3) for d in range(3)]
    raise ValueError(cfg.kind)


def assemble_blocks(cfg, blocks: dict[str, np.ndarray], E: int) -> np.ndarray:
    """Per-block outputs A{c}{d}[E][ns][ns] -> A[E][3ns][3ns] (component-blocked)."""
    if "A" in blocks:
        return blocks["A"].reshape(E, cfg.n, cfg.n)
    ns = cfg.ns
    A = np.zeros((E, 3 * ns, 3 * ns))
    for c in range(3):
        for d in range(3):
            A[:, c * ns:(c + 1) * ns, d * ns:(d + 1) * ns] = blocks[f"A{c}{d}"].reshape(E, ns, ns)
    return A


def argument_order(ir: dict):
    """(outputs, input tables, constants) in emitted-C order (emit_c.cpp:137-140)."""
    outs = sorted(ir["outputs"])
    tabs = sorted(n for n, t in ir["tables"].items() if t.get("provenance", "input") == "input")
    consts = sorted(ir.get("constants", {}))
    return outs, tabs, consts


def e_tables(cfg, coords, coeffs) -> dict:
    """The per-cell (SoA, ``name[e]``) input tables of this module's IR for a whole
    mesh, from cell-major coords ``[E][4][3]`` and coefficients ``[E][ncoef]``:
    what a caller supplies at run time to a kernel built on a few cells."""
    coords = np.asarray(coords, dtype=np.float64)
    coeffs = np.asarray(coeffs, dtype=np.float64)
    E = coords.shape[0]
    x = coords.reshape(E, 4, 3)
    t = {f"x{v}{c}": x[:, v, c] for v in range(4) for c in range(3)}
    ns = cfg.ns
    if cfg.kind == fe.HELMHOLTZ:
        t.update({f"f{m:02d}": coeffs[:, m] for m in range(coeffs.shape[1])})
    elif cfg.kind == fe.ELASTICITY:
        t.update({f"mu{m}": coeffs[:, m] for m in range(4)})
        t.update({f"lam{m}": coeffs[:, 4 + m] for m in range(4)})
    elif cfg.kind == fe.HYPERELASTICITY:
        t.update({f"w{c}{m:02d}": coeffs[:, c * ns + m] for c in range(3) for m in range(ns)})
        t.update({f"mu{m}": coeffs[:, 3 * ns + m] for m in range(4)})
        t.update({f"lam{m}": coeffs[:, 3 * ns + 4 + m] for m in range(4)})
    else:
        t.update({f"u{c}{m:02d}": coeffs[:, c * ns + m] for c in range(3) for m in range(ns)})
    return {k: np.ascontiguousarray(v) for k, v in t.items()}


def dumps(ir: dict) -> str:
    return json.dumps(ir, separators=(",", ":"))
