"""Published step tables for the k-bit activations (product-side copy of the
paper's constants; the oracle keeps its own).  Levels are the cumulative ReLU
weights of Eq. 14: s = (0, a1, a1 + a2, 1)."""

# ReGELU2, App. E
REGELU2 = dict(act="gelu", k=2, a=(-0.04922261145617846, 1.0979632065417297),
               c=(-3.1858810036855245, -0.001178821281161997, 3.190832613414926))
# ReSiLU2, App. E
RESILU2 = dict(act="silu", k=2, a=(-0.04060357190528599, 1.080925428529668),
               c=(-6.3050461001646445, -0.0008684942046214787, 6.325815242089708))
# ReGELU2-d, App. I: derivative-L2 objective
REGELU2_D = dict(act="gelu", k=2, a=(0.32465931184406527, 0.34812875668739607),
                 c=(-0.4535743722857079, -0.0010587205574873046, 0.4487575313884231))


def levels(table):
    """s_j = sum of the first j weights of Eq. 14, the last
    weight being 1 - sum(a), so s_0 = 0 and s_m = 1 exactly; for k = 2 this is
    (0, a1, a1 + a2, 1).  Requires the thresholds sorted increasingly (the
    fitter's canonical order, DESIGN F5)."""
    a = [float(v) for v in table["a"]]
    out, acc = [0.0], 0.0
    for w in a:
        acc += w
        out.append(acc)
    out.append(1.0)
    return tuple(out)


def from_fit(f):
    """Step table of a fitter result (fit.Fit: a = m - 1 weights, c = m
    thresholds, m = 2^k - 1, pairs sorted by c)."""
    c = [float(v) for v in f.c]
    if sorted(c) != c:
        raise ValueError("fitter thresholds must be increasing")
    return dict(act=f.act, k=f.k, a=tuple(f.a), c=tuple(c))
