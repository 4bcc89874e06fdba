"""Graph cases for deduction parity (tests/test_graph_parity.py).

Seeded random CompGraphs in the line form of include/hshard/graph.hpp --
placeholders / parameters with literal and symbolic dims, Elementwise, Dot,
Sum, Reshape (merge / split dims) and CommOps -- with random leaf / CommOp
annotations per strategy, biased towards ones that deduce (shared device
groups, 1-3 subgroups, Split / Duplicate / Partial keys, top-tier splits with
ratios), plus hand-written cases for each rule and error path.  f32 / f64
only: the reference DType has no bf16.
"""
import random

DIMS = [4, 8, 12, 16, "B", "2*B", "B/2", "S"]


def _factorizations(n):
    if n == 1:
        return [[]]
    out = []
    for f in range(2, n + 1):
        if n % f == 0:
            for rest in _factorizations(n // f):
                out.append([f] + rest)
    return out


def _ds(rng, n, rank):
    counts = rng.choice(_factorizations(n)) if n > 1 else []
    keys = [-1, -2] + list(range(rank))
    ent = []
    for c in counts:
        k = rng.choice(keys)
        if rng.random() < 0.35:
            k = -1
        ent.append((k, c))
    return "{" + ",".join(f"{k}:{c}" for k, c in ent) + "}"


def _groups(rng):
    devs = list(range(8))
    rng.shuffle(devs)
    h = rng.choice([1, 1, 2, 2, 3])
    sizes = {1: [[2], [4], [1], [8]], 2: [[2, 2], [4, 4], [4, 2], [2, 1]], 3: [[2, 1, 1], [4, 2, 2], [2, 2, 2]]}[h]
    sz = rng.choice(sizes)
    out, i = [], 0
    for s in sz:
        out.append(sorted(devs[i:i + s]))
        i += s
    return out


def _anno(rng, groups, rank):
    h = len(groups)
    specs = [_ds(rng, len(g), rank) for g in groups]
    body = "; ".join("(" + ",".join(map(str, g)) + ")" + s for g, s in zip(groups, specs))
    if h == 1:
        return f"hsize=1 hdim=-1 [{body}]"
    hdim = rng.choice([-1, -2] + list(range(rank)))
    ratios = ""
    if hdim >= 0 and rng.random() < 0.4:
        ratios = " ratios=" + ",".join(["1/2", "1/4", "1/4"][:h] if h == 3 else ["3/4", "1/4"])
    return f"hsize={h} hdim={hdim} [{body}]{ratios}"


def random_graph(seed):
    rng = random.Random(seed)
    nstrat = rng.choice([1, 2, 3])
    lines = [f"strategies {nstrat}"]
    shapes, leaves, comms = [], [], []
    dtype = rng.choice(["f32", "f64"])
    base_groups = [_groups(rng) for _ in range(nstrat)]

    def add(stmt, shape):
        lines.append(stmt)
        shapes.append(shape)
        return len(shapes) - 1

    def leaf(kind):
        rank = rng.choice([1, 2, 2, 3])
        shape = [rng.choice(DIMS) for _ in range(rank)]
        t = add(f"{kind} {kind[0]}{len(shapes)} {dtype} " + " ".join(map(str, shape)), shape)
        leaves.append(t)
        return t

    live = [leaf("placeholder"), leaf("parameter")]
    for _ in range(rng.randint(1, 7)):
        op = rng.choice(["ew", "dot", "dot", "sum", "reshape", "comm", "param"])
        x = rng.choice(live)
        sx = shapes[x]
        if op == "ew":
            live.append(add(f"elementwise {rng.choice(['identity', 'relu', 'gelu'])} {x}", sx))
        elif op == "dot":
            k = rng.choice(DIMS)
            w = add(f"parameter w{len(shapes)} {dtype} {sx[-1]} {k}", [sx[-1], k])
            leaves.append(w)
            live.append(add(f"dot {x} {w}", sx[:-1] + [k]))
        elif op == "sum" and len(sx) > 1:
            a = rng.randrange(len(sx))
            live.append(add(f"sum {x} {a}", sx[:a] + sx[a + 1:]))
        elif op == "reshape":
            lit = [d for d in sx if isinstance(d, int)]
            if len(sx) >= 2 and all(isinstance(d, int) for d in sx[:2]):
                tgt = [sx[0] * sx[1]] + sx[2:]
            elif lit and lit[0] % 2 == 0:
                i = sx.index(lit[0])
                tgt = sx[:i] + [2, lit[0] // 2] + sx[i + 1:]
            elif sx[0] == "B":
                tgt = ["B/2", 2] + sx[1:]
            else:
                tgt = sx[::-1]
            live.append(add(f"reshape {x} " + " ".join(map(str, tgt)), tgt))
        elif op == "comm":
            t = add(f"comm {x} {rng.choice(['auto', '0', '1'])}", sx)
            comms.append(t)
            live.append(t)
        elif op == "param":
            live.append(leaf("parameter"))
    for s in range(nstrat):
        for t in leaves + comms:
            groups = base_groups[s] if rng.random() < 0.85 else _groups(rng)
            if rng.random() < 0.03:
                continue  # an unannotated leaf: UndeducedStrategy
            lines.append(f"annotate {t} {s} {_anno(rng, groups, len(shapes[t]))}")
    return "\n".join(lines)


def handwritten():
    g = []
    # Megatron MLP: x Dup, w1 col-split, gelu, w2 row-split -> Partial, AllReduce CommOp
    g.append("\n".join([
        "strategies 2",
        "placeholder x f32 B 64", "parameter w1 f32 64 256", "dot 0 1", "elementwise gelu 2",
        "parameter w2 f32 256 64", "dot 3 4", "comm 5 auto",
        "annotate 0 0 hsize=1 hdim=-1 [(0,1,2,3){-1:4}]", "annotate 1 0 hsize=1 hdim=-1 [(0,1,2,3){1:4}]",
        "annotate 4 0 hsize=1 hdim=-1 [(0,1,2,3){0:4}]", "annotate 6 0 hsize=1 hdim=-1 [(0,1,2,3){-1:4}]",
        "annotate 0 1 hsize=1 hdim=-1 [(0,1,2,3){0:2,-1:2}]", "annotate 1 1 hsize=1 hdim=-1 [(0,1,2,3){-1:2,1:2}]",
        "annotate 4 1 hsize=1 hdim=-1 [(0,1,2,3){-1:2,0:2}]", "annotate 6 1 hsize=1 hdim=-1 [(0,1,2,3){0:2,-1:2}]"]))
    # heterogeneous DP: two subgroups, batch split 3:1 across them
    g.append("\n".join([
        "strategies 1", "placeholder x f64 B 32", "parameter w f64 32 16", "dot 0 1", "sum 2 0",
        "annotate 0 0 hsize=2 hdim=0 [(0,1){-1:2}; (2,3){-1:2}] ratios=3/4,1/4",
        "annotate 1 0 hsize=2 hdim=-1 [(0,1){-1:2}; (2,3){-1:2}]"]))
    # contraction split across subgroups: equal ratios required (ok) / differing (error)
    for r in ["1/2,1/2", "3/4,1/4"]:
        g.append("\n".join([
            "strategies 1", "placeholder x f32 8 16", "parameter w f32 16 8", "dot 0 1",
            "annotate 0 0 hsize=2 hdim=1 [(0,1){-1:2}; (2,3){-1:2}] ratios=1/2,1/2",
            f"annotate 1 0 hsize=2 hdim=0 [(0,1){{-1:2}}; (2,3){{-1:2}}] ratios={r}"]))
    # reshapes: merge, split, symbolic, and a split that does not survive
    g.append("\n".join([
        "strategies 1", "placeholder x f32 B 4 8", "reshape 0 B 32", "reshape 1 B/2 2 32",
        "annotate 0 0 hsize=1 hdim=-1 [(0,1){0:2}]"]))
    g.append("\n".join([
        "strategies 1", "placeholder x f32 4 8", "reshape 0 32",
        "annotate 0 0 hsize=1 hdim=-1 [(0,1){1:2}]"]))
    # unification across hsize (convert_hsize) and a DG mismatch needing a CommOp
    g.append("\n".join([
        "strategies 2", "placeholder x f32 8 8", "parameter w f32 8 8", "dot 0 1",
        "annotate 0 0 hsize=1 hdim=-1 [(0,1,2,3){-1:4}]", "annotate 1 0 hsize=2 hdim=-1 [(0,1){1:2}; (2,3){1:2}]",
        "annotate 0 1 hsize=1 hdim=-1 [(0,1){-1:2}]", "annotate 1 1 hsize=1 hdim=-1 [(2,3){1:2}]"]))
    # both operands Partial, an out-of-range split dim, a missing annotation
    g.append("\n".join([
        "strategies 3", "placeholder x f32 8 8", "parameter w f32 8 8", "dot 0 1",
        "annotate 0 0 hsize=1 hdim=-1 [(0,1){-2:2}]", "annotate 1 0 hsize=1 hdim=-1 [(0,1){-2:2}]",
        "annotate 0 1 hsize=1 hdim=-1 [(0,1){5:2}]", "annotate 1 1 hsize=1 hdim=-1 [(0,1){-1:2}]",
        "annotate 0 2 hsize=1 hdim=-1 [(0,1){-1:2}]"]))
    # pipelines: a forward hand-off 0 -> 1 and a second one back 1 -> 0 make
    # device 1 both one stage after and one stage before device 0
    # (ConflictingStageOrder); a plain 0 -> 1 -> 2 chain is three stages
    g.append("\n".join([
        "strategies 2", "placeholder x f32 8 8", "comm 0 0", "elementwise relu 1", "comm 2 0",
        "annotate 0 0 hsize=1 hdim=-1 [(0){}]", "annotate 1 0 hsize=1 hdim=-1 [(1){}]",
        "annotate 3 0 hsize=1 hdim=-1 [(0){}]",
        "annotate 0 1 hsize=1 hdim=-1 [(0){}]", "annotate 1 1 hsize=1 hdim=-1 [(1){}]",
        "annotate 3 1 hsize=1 hdim=-1 [(2){}]"]))
    return g


def all_cases(n_random=300):
    return handwritten() + [random_graph(1000 + i) for i in range(n_random)]
