"""Case generators for the golden fixtures (ref_tool line protocol, see
oracle/ref_tool.cpp).  Shared by make_golden.py (which runs the reference)
and by the tests (which replay the same commands through the product)."""
from __future__ import annotations

import os
import random
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def A(groups, specs, hdim=-1, ratios=None):
    parts = ["(" + ",".join(map(str, g)) + ")" + s for g, s in zip(groups, specs)]
    s = f"hsize={len(groups)} hdim={hdim} [" + "; ".join(parts) + "]"
    if ratios:
        s += " ratios=" + ",".join(ratios)
    return s


def S(group, spec):
    return A([group], [spec], -1)


def sh(shape):
    return ",".join(str(x) for x in shape)


def C(src, dst, shape, dtype="f32", bw="u"):
    return [f"C|{dtype}|{sh(shape)}|{bw}|{src}|{dst}"]


def kat_commands():
    q = [0, 1, 2, 3]
    cmds = []
    # Fig 6 bottom-tier table
    cmds += C(S(q, "{-2:4}"), S(q, "{-1:4}"), [8, 8])
    cmds += C(S(q, "{-2:4}"), S(q, "{0:4}"), [8, 8])
    cmds += C(S(q, "{0:4}"), S(q, "{-1:4}"), [8, 8])
    cmds += C(S(q, "{0:2,-1:2}"), S(q, "{0:4}"), [8, 8])
    cmds += C(S(q, "{0:4}"), S(q, "{0:4}"), [8, 8])                      # Identity
    cmds += C(S(q, "{0:4}"), S([4, 5, 6, 7], "{0:4}"), [8, 8])           # SendRecv
    cmds += C(S(q, "{0:4}"), S([0, 1, 2, 4], "{0:4}"), [8, 8])           # SR self-pairs
    cmds += C(S([3, 1, 0, 2], "{-2:4}"), S([3, 1, 0, 2], "{0:4}"), [8, 8])  # RS group order
    cmds += C(S(q, "{-2:4}"), S([0, 1], "{0:2}"), [8, 8])                # PartialUnderBsr
    cmds += C(S(q, "{0:4}"), S([0, 1], "{0:2}"), [8, 8])                 # hsize/DG change -> Bsr
    # top tier
    d2 = [[0, 1], [2, 3]]
    cmds += C(A(d2, ["{0:2}", "{0:2}"], -2), A(d2, ["{0:2}", "{0:2}"], -1), [8, 8])
    cmds += C(A(d2, ["{1:2}", "{1:2}"], 0), A(d2, ["{1:2}", "{1:2}"], -1), [8, 8])
    cmds += C(A(d2, ["{0:2}", "{0:2}"], -2), A(d2, ["{1:2}", "{1:2}"], 0), [8, 8])
    cmds += C(A(d2, ["{0:2}", "{0:2}"], -2), A(d2, ["{0:2}", "{0:2}"], 0), [8, 8])
    cmds += C(A(d2, ["{0:2}", "{0:2}"], 0), A(d2, ["{0:2}", "{0:2}"], -2), [8, 8])  # unsupported -> Bsr/err
    # Appendix B1 defect repros (planner parity must reproduce them)
    cmds += C(S([3, 5, 2, 7], "{1:4}"), S([3, 5, 2, 7], "{-1:2,1:2}"), [12, 4])
    cmds += C(S([2, 5, 6, 4], "{-2:2,0:2}"), S([2, 5, 6, 4], "{0:4}"), [16, 8])
    cmds += C(S(list(range(6)), "{-2:2,1:3}"), S(list(range(6)), "{1:6}"), [4, 12])
    # placement / convert_hsize / equality / alignment / validate
    cmds += [f"P|8,2|{S(q, '{0:4}')}"]
    cmds += [f"P|4,4|{A([[0, 1], [2]], ['{1:2}', '{-1:1}'], 0, ['1/2', '1/2'])}"]
    cmds += [f"P|4096,4096|{A(d2, ['{-1:2}', '{-1:2}'], 0, ['3/4', '1/4'])}"]
    cmds += [f"H|{A([q], ['{0:4}'], 0)}|2", f"H|{S(q, '{-1:4}')}|4", f"H|{A([[0, 1, 2]], ['{0:3}'], 0)}|2"]
    cmds += [f"Q|{S([0, 1], '{0:2,-1:1}')}|{S([0, 1], '{0:2}')}", f"Q|{S(q, '{0:4}')}|{A([q], ['{0:4}'], 0)}"]
    cmds += ["A|{0:2,-1:2}|{0:4}", "A|{1:4}|{-1:2,1:2}", "A|{0:2,1:3}|{1:3,0:2}", "A|{0:4}|{-1:2}"]
    cmds += [f"V|8|{S(q, '{0:3}')}", f"V|8|{A([[0, 1], [1, 2]], ['{0:2}', '{0:2}'])}",
             f"V|8|{S(q, '{0:2,-1:2}')}", f"V|6|{S(q, '{0:4}')}"]
    # BSR table / heuristics
    cmds += [f"T|4|8|0|{S([0, 1], '{0:2}')}|{S(q, '{0:4}')}"]
    cmds += [f"T|4|4|3|{S([0, 1], '{-1:2}')}|{S([0, 1], '{0:2}')}"]
    cmds += [f"M|d=1;8-9=2|0|4|4|{S([1, 9], '{-1:2}')}|{S([8], '{}')}"]   # heuristic II -> 9
    cmds += [f"M|u|0|4|4|{S([1, 2], '{-1:2}')}|{S([0, 3], '{0:2}')}"]      # heuristic III -> 1, 2
    cmds += [f"M|u|1|4|4|{S([1, 2], '{-1:2}')}|{S([0, 3], '{0:2}')}"]      # naive -> 1, 1
    cmds += [["F|u|2", f"0|4|8|{S([0], '{}')}|{S([1], '{}')}", f"1|4|8|{S([0], '{}')}|{S([1], '{}')}"]]
    cmds += [["F|u|1", f"5|4|4|{S([0, 1], '{-1:2}')}|{S([2, 3], '{-1:2}')}"]]
    return [c if isinstance(c, list) else [c] for c in cmds]


def workload_commands():
    from paper_2504_20490_b200 import workloads as W
    cmds = []
    for w in W.all_workloads():
        if w.kind == "classify":
            for tid, src, dst, shape in w.transitions:
                dt = "f32" if w.dtype == "bf16" else w.dtype  # the reference has no bf16
                cmds.append(C(src, dst, shape, dt))
        else:
            lines = [f"F|u|{len(w.transitions)}"]
            for tid, src, dst, shape in w.transitions:
                lines.append(f"{tid}|2|{sh(shape)}|{src}|{dst}")
            cmds.append(lines)
    return cmds


# ---------------------------------------------------------------- random sweep
KEYS = [-2, -1, 0, 1]


def _factorizations(n, rng):
    fs = []
    while n > 1:
        ds = [d for d in range(2, n + 1) if n % d == 0]
        d = rng.choice(ds)
        fs.append(d)
        n //= d
    rng.shuffle(fs)
    return fs


def rand_ds(rng, n, ndim, allow_partial=True, allow_dup=True):
    keys = [k for k in KEYS if (k >= 0 and k < ndim) or (k == -2 and allow_partial) or
            (k == -1 and allow_dup)]
    for _ in range(20):
        fs = _factorizations(n, rng)
        if len(fs) <= len(keys):
            break
    else:
        fs = [n] if n > 1 else []
    ks = rng.sample(keys, len(fs))
    ents = list(zip(ks, fs))
    # unit entry with a key not used elsewhere (keys must stay unique)
    used = {k for k, _ in ents}
    free = [k for k in keys if k not in used]
    if free and rng.random() < 0.1:
        ents.insert(rng.randrange(len(ents) + 1), (rng.choice(free), 1))
    return "{" + ",".join(f"{k}:{c}" for k, c in ents) + "}"


def rand_ratios(rng, h):
    den = rng.choice([2, 3, 4, 8])
    if den < h:
        den = h * 2
    cuts = sorted(rng.sample(range(1, den), h - 1))
    parts = [b - a for a, b in zip([0] + cuts, cuts + [den])]
    return [str(Fraction(p, den)) if Fraction(p, den).denominator != 1 else "1" for p in parts]


def rand_groups(rng, devs, hsize):
    devs = list(devs)
    rng.shuffle(devs)
    cuts = sorted(rng.sample(range(1, len(devs)), hsize - 1)) if hsize > 1 else []
    return [devs[a:b] for a, b in zip([0] + cuts, cuts + [len(devs)])]


def rand_anno(rng, groups, ndim, allow_partial=True, hdim=None):
    h = len(groups)
    if hdim is None:
        hdim = rng.choice([-2, -1] + list(range(ndim)) if allow_partial else [-1] + list(range(ndim)))
    specs = [rand_ds(rng, len(g), ndim, allow_partial) for g in groups]
    ratios = rand_ratios(rng, h) if (hdim >= 0 and h > 1 and rng.random() < 0.5) else None
    return A(groups, specs, hdim, ratios)


def zero_width(text, shape):
    """True when a top-tier ratio slice floors to zero width (reference UB, App. B3)."""
    from paper_2504_20490_b200.hshard import parse_annotation
    a = parse_annotation(text)
    h, hd = a["hsize"], a["hdim"]
    if h == 1 or hd < 0 or hd >= len(shape):
        return False
    ratios = a["ratios"] or [Fraction(1, h)] * h
    cum, bounds = Fraction(0), [0]
    for r in ratios[:-1]:
        cum += r
        bounds.append((cum * shape[hd]).__floor__())
    bounds.append(shape[hd])
    return any(b <= a_ for a_, b in zip(bounds, bounds[1:]))


def rand_pair(rng, partial_ok=True):
    """Random (src, dst, shape) biased towards executable plans of every kind."""
    ndim = rng.choice([1, 2, 2])
    shape = [rng.choice([8, 12, 16, 24]) for _ in range(ndim)]
    pool = rng.sample(range(10), rng.randint(1, 8))
    hs = rng.choice([1, 1, 2, 2, 3]) if len(pool) >= 3 else rng.choice([1, len(pool)])
    hs = min(hs, len(pool))
    groups = rand_groups(rng, pool, hs)
    mode = rng.random()
    if mode < 0.35:      # branch (a): same DG union and top tier
        hdim = rng.choice(([-2] if partial_ok else []) + [-1] + list(range(ndim)))
        src = rand_anno(rng, groups, ndim, partial_ok, hdim=hdim)
        ratios = src.split(" ratios=")[1].split(",") if " ratios=" in src else None
        dst = A(groups, [rand_ds(rng, len(g), ndim, partial_ok) for g in groups], hdim, ratios)
    elif mode < 0.6 and partial_ok and hs > 1:   # branch (b): split collectives
        d = rng.randrange(ndim)
        h0, h1 = rng.choice([(-2, -1), (-2, d), (d, -1)])
        sspecs = [rand_ds(rng, len(g), ndim, True) for g in groups]
        dspecs = sspecs if rng.random() < 0.5 else [rand_ds(rng, len(g), ndim, True) for g in groups]
        r0 = rand_ratios(rng, hs) if h0 >= 0 and rng.random() < 0.5 else None
        r1 = rand_ratios(rng, hs) if h1 >= 0 and rng.random() < 0.5 else None
        src, dst = A(groups, sspecs, h0, r0), A(groups, dspecs, h1, r1)
    elif mode < 0.8:     # branch (c): unrelated, Partial-free
        src = rand_anno(rng, groups, ndim, False)
        pool2 = rng.sample(range(10), rng.randint(1, 8))
        hs2 = min(rng.choice([1, 1, 2, 3]), len(pool2))
        dst = rand_anno(rng, rand_groups(rng, pool2, hs2), ndim, False)
    elif mode < 0.9:     # Identity / SendRecv
        src = rand_anno(rng, groups, ndim, partial_ok)
        if rng.random() < 0.5:
            dst = src
        else:
            p = parse_groups(src)
            perm = rng.sample(range(10), sum(len(g) for g in p))
            it = iter(perm)
            dst = src.split("[")[0] + "[" + "; ".join(
                "(" + ",".join(str(next(it)) for _ in g) + ")" + "{" + part.split("{", 1)[1]
                for g, part in zip(p, src.split("[", 1)[1].rsplit("]", 1)[0].split(";"))) + "]" + \
                src.rsplit("]", 1)[1]
    else:                # anything
        src = rand_anno(rng, groups, ndim, partial_ok)
        pool2 = rng.sample(range(10), rng.randint(1, 8))
        hs2 = min(rng.choice([1, 1, 2, 3]), len(pool2))
        dst = rand_anno(rng, rand_groups(rng, pool2, hs2), ndim, partial_ok and rng.random() < 0.3)
    return src, dst, shape


def parse_groups(text):
    body = text[text.index("[") + 1:text.rindex("]")]
    return [[int(x) for x in part[part.index("(") + 1:part.index(")")].split(",") if x.strip()]
            for part in body.split(";")]


def random_commands(seed, n):
    rng = random.Random(seed)
    cmds = []
    while len(cmds) < n:
        r = rng.random()
        src, dst, shape = rand_pair(rng)
        if zero_width(src, shape) or zero_width(dst, shape):
            continue
        if r < 0.62:
            dt = rng.choice(["f32", "f64", "i32", "i64"])
            bw = "u" if rng.random() < 0.7 else "d=1;" + ";".join(
                f"{a}-{b}={rng.choice([2, 3])}" for a, b in
                (rng.sample(range(10), 2) for _ in range(rng.randint(1, 6))))
            cmds.append(C(src, dst, shape, dt, bw))
        elif r < 0.72:
            cmds.append([f"T|{rng.choice([2, 4, 8])}|{sh(shape)}|{rng.randrange(5)}|{src}|{dst}"])
        elif r < 0.82:
            bw = "u" if rng.random() < 0.5 else "d=1;" + ";".join(
                f"{a}-{b}=2" for a, b in (rng.sample(range(10), 2) for _ in range(3)))
            cmds.append([f"M|{bw}|{int(rng.random() < 0.3)}|4|{sh(shape)}|{src}|{dst}"])
        elif r < 0.87:
            k = rng.randint(2, 4)
            lines = [f"F|u|{k}"]
            for t in range(k):
                s2, d2, shp = rand_pair(rng, partial_ok=False)
                if zero_width(s2, shp) or zero_width(d2, shp):
                    s2, d2, shp = S([0, 1], "{-1:2}"), S([2, 3], "{0:2}"), [8]
                lines.append(f"{t * 3 + 1}|4|{sh(shp)}|{s2}|{d2}")
            cmds.append(lines)
        elif r < 0.92:
            cmds.append([f"P|{sh(shape)}|{src}"])
        elif r < 0.95:
            cmds.append([f"H|{src}|{rng.choice([2, 3, 4, 6])}"])
        elif r < 0.97:
            cmds.append([f"Q|{src}|{dst if rng.random() < 0.5 else src}"])
        else:
            cmds.append([f"V|{sh(shape)}|{src}"])
    return cmds


def random_exec_commands(seed, n):
    rng = random.Random(seed)
    cmds = []
    while len(cmds) < n:
        src, dst, shape = rand_pair(rng)
        if zero_width(src, shape) or zero_width(dst, shape):
            continue
        dt = rng.choice(["f32", "f64", "i32", "i64"])
        cmds.append([f"X|{dt}|{sh(shape)}|u|{src}|{dst}|{rng.randrange(1000)}|grid|1|1"])
    return cmds
