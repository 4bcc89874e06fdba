"""Records the reference volume_report (bsr.hpp:107-108, bsr.cpp:244-261) of fused
switch plans through oracle/_ref/ref_tool (command R) into tests/golden/volume.jsonl.
Run in a container that has /root/reference (the oracle build); the fixture is
committed so the GPU box and CPU tests replay it without the reference."""
import json
import os
import random
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from gen_cases import rand_pair  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def cases():
    from paper_2504_20490_b200 import workloads as W
    out = []
    w = W.config4()
    out.append(("cfg4", [(t, 2, list(sh), s, d) for t, s, d, sh in w.transitions],
                {d: d // 4 for d in range(8)}))
    out.append(("cfg4-8pernode", [(t, 2, list(sh), s, d) for t, s, d, sh in w.transitions],
                {d: 0 for d in range(8)}))
    rng = random.Random(5)
    ok = err = 0
    while ok < 40:
        ents = []
        for tid in range(rng.randint(1, 4)):
            src, dst, shape = rand_pair(rng)
            ents.append((tid, 4, shape, src, dst))
        node_of = {d: rng.randint(0, 2) for d in range(12)}
        res = run(ents, node_of)
        if "error" in res:
            if err >= 5:
                continue
            err += 1
        else:
            ok += 1
        out.append((f"rand{ok}_{err}", ents, node_of))
    # a transfer end outside the cluster map
    out.append(("unknown-device", out[0][1], {d: 0 for d in range(4)}))
    return out


def run(ents, node_of, bw="u"):
    cmd = f"R|{bw}|{len(ents)}|" + ",".join(f"{d}:{n}" for d, n in sorted(node_of.items())) + "\n"
    for tid, eb, shape, src, dst in ents:
        cmd += f"{tid}|{eb}|{','.join(map(str, shape))}|{src}|{dst}\n"
    res = subprocess.run([REF], input=cmd, capture_output=True, text=True, timeout=600)
    return json.loads(res.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    with open(os.path.join(HERE, "volume.jsonl"), "w") as f:
        for name, ents, node_of in cases():
            f.write(json.dumps({"name": name, "entries": ents, "node_of": node_of, "out": run(ents, node_of)}) + "\n")
    print("wrote", os.path.join(HERE, "volume.jsonl"))
