"""Generate hpg_usmall_gen.cuh: straight-line U-side code per low degree p.

For p <= PMAX the per-cell U-side work of the residual (
hpgalerkin/assembly.py:42-116, 470-477, 725-729) is written out as explicit
FMA sequences with literal reference-cell coefficients:

  A u      = (hy/hx) (Kref C Mref) + (hx/hy) (Mref C Kref)
  B dpsi   = R^T G R                      (obstacle)
           = D^T Gx R + R^T Gy D           (gradient)
  B^T u    = wx (R C R^T) wy               (obstacle)
           = [w2 (D C R^T) wy ; wx (R C D^T) w2]   (gradient)

R: U dof -> Legendre map (spaces.py:45-57), D: derivative map (:59-68),
Kref = h * local stiffness, Mref = R^T diag(1/(2l+1)) R = local mass / h.
Coefficients are exact rationals evaluated in fp64 here.  C and G are any
indexable operands (shared-memory slices in k_usmall, lazy global-memory
accessors in k_lowp, where dead outputs and their loads are eliminated).

    python tools/gen_usmall.py        (rewrites the header)
"""
import os
from fractions import Fraction as F

PMAX = 8
OUT = os.path.join(os.path.dirname(__file__), "..", "paper_2412_13733_b200", "csrc",
                   "hpg_usmall_gen.cuh")


def R(p):
    m = p + 1
    r = [[F(0)] * m for _ in range(m)]
    r[0][0] = F(1, 2); r[1][0] = F(-1, 2); r[0][1] = F(1, 2); r[1][1] = F(1, 2)
    for q in range(p - 1):
        r[q][2 + q] = F(1, 2 * q + 3)
        r[q + 2][2 + q] = F(-1, 2 * q + 3)
    return r


def D(p):
    m = p + 1
    d = [[F(0)] * m for _ in range(max(p, 1))]
    d[0][0] = F(-1, 2); d[0][1] = F(1, 2)
    for q in range(p - 1):
        d[q + 1][2 + q] = F(-1)
    return d


def Kref(p):
    m = p + 1
    k = [[F(0)] * m for _ in range(m)]
    k[0][0] = F(1); k[0][1] = F(-1); k[1][0] = F(-1); k[1][1] = F(1)
    for q in range(p - 1):
        k[2 + q][2 + q] = F(4, 2 * q + 3)
    return k


def Mref(p):
    m = p + 1
    r = R(p)
    return [[sum(r[l][a] * r[l][b] / (2 * l + 1) for l in range(m)) for b in range(m)]
            for a in range(m)]


def lit(x):
    return repr(float(x))


def gen(p, gradient):
    m = p + 1
    n = p if gradient else p - 1
    r, d, k, mm = R(p), D(p), Kref(p), Mref(p)
    lines = []
    w = lines.append
    w(f"template <> struct USmall<{p}, {'true' if gradient else 'false'}> {{")
    w("template <class CA, class GA, class OU, class OB>")
    w("__device__ __forceinline__ static void run(")
    w("    const CA& C, const GA& G, int TH, double hx, double hy,")
    w("    double alpha, OU ou, OB ob) {")
    w(f"  // p = {p}: m = {m}, n = {n}; C[(i*{m}+l)*TH], G[((comp*{n}+i)*{n}+l)*TH] (raw psi_prev - psi)")
    w("  const double sKM = hy / hx, sMK = hx / hy;")
    # A u + B dpsi -> rloc[j*m+k]
    for j in range(m):
        for kk in range(m):
            t1 = []   # Kref (x) Mref
            t2 = []   # Mref (x) Kref
            for jp in range(m):
                for kp in range(m):
                    c1 = k[j][jp] * mm[kk][kp]
                    c2 = mm[j][jp] * k[kk][kp]
                    if c1 != 0:
                        t1.append((c1, jp * m + kp))
                    if c2 != 0:
                        t2.append((c2, jp * m + kp))
            e1 = " + ".join(f"{lit(c)} * C[{ix} * TH]" for c, ix in t1) or "0.0"
            e2 = " + ".join(f"{lit(c)} * C[{ix} * TH]" for c, ix in t2) or "0.0"
            # B dpsi
            tb = []
            comps = (0, 1) if gradient else (0,)
            for comp in comps:
                for i in range(n):
                    for l in range(n):
                        if not gradient:
                            a = r[i][j] * r[l][kk] / ((2 * i + 1) * (2 * l + 1))
                            sc = "hx * hy"
                        elif comp == 0:
                            a = (d[i][j] if i < len(d) else 0) * r[l][kk] * F(2, 2 * i + 1) / (2 * l + 1)
                            sc = "hy"
                        else:
                            a = r[i][j] * (d[l][kk] if l < len(d) else 0) / (2 * i + 1) * F(2, 2 * l + 1)
                            sc = "hx"
                        if a != 0:
                            tb.append((a, comp * n * n + i * n + l, sc))
            if not gradient:
                eb = " + ".join(f"{lit(a)} * G[{ix} * TH]" for a, ix, _ in tb)
                eb = f"(hx * hy) * ({eb})" if eb else "0.0"
            else:
                ex = " + ".join(f"{lit(a)} * G[{ix} * TH]" for a, ix, sc in tb if sc == "hy")
                ey = " + ".join(f"{lit(a)} * G[{ix} * TH]" for a, ix, sc in tb if sc == "hx")
                parts = []
                if ex:
                    parts.append(f"hy * ({ex})")
                if ey:
                    parts.append(f"hx * ({ey})")
                eb = " + ".join(parts) or "0.0"
            w(f"  ou({j}, {kk}, -alpha * (sKM * ({e1}) + sMK * ({e2})) + ({eb}));")
    # B^T u -> btu[(comp*n+a)*n+b]
    for comp in ((0, 1) if gradient else (0,)):
        for a in range(n):
            for b in range(n):
                terms = []
                for i in range(m):
                    for l in range(m):
                        if not gradient:
                            c = r[a][i] * r[b][l] / ((2 * a + 1) * (2 * b + 1))
                        elif comp == 0:
                            c = d[a][i] * r[b][l] * F(2, 2 * a + 1) / (2 * b + 1)
                        else:
                            c = r[a][i] * d[b][l] / (2 * a + 1) * F(2, 2 * b + 1)
                        if c != 0:
                            terms.append((c, i * m + l))
                e = " + ".join(f"{lit(c)} * C[{ix} * TH]" for c, ix in terms) or "0.0"
                sc = "hx * hy" if not gradient else ("hy" if comp == 0 else "hx")
                w(f"  ob({comp}, {a}, {b}, ({sc}) * ({e}));")
    w("}")
    w("};")
    return "\n".join(lines)


def main():
    parts = ["// GENERATED by tools/gen_usmall.py -- do not edit.",
             "// Straight-line per-cell U-side code for p <= %d (see the generator's docstring)." % PMAX,
             "#pragma once", "namespace hpg {",
             "template <int P, bool GRADIENT> struct USmall;",
             f"constexpr int USMALL_PMAX = {PMAX};"]
    for p in range(2, PMAX + 1):
        parts.append(gen(p, False))
    for p in range(1, PMAX + 1):
        parts.append(gen(p, True))
    parts.append("}  // namespace hpg\n")
    with open(OUT, "w") as f:
        f.write("\n".join(parts))
    print("wrote", OUT, os.path.getsize(OUT) // 1024, "KB")


if __name__ == "__main__":
    main()
