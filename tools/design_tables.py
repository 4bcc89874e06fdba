"""Regenerates DESIGN.md's graph-switch tables (N=1 cold/warm per step, N=2/N=4
cold/warm/tuned and pipelined cycles) from the committed bench lines in profiles/."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {'cfg4': 'cfg4 TP2×PP4 → TP4×PP2', 'cfg4_rev': 'cfg4 reverse', 'cfg5_S1S2': 'cfg5 S1→S2',
         'cfg5_S2S3': 'cfg5 S2→S3', 'cfg5_S3S4': 'cfg5 S3→S4', 'cfg5_S4S1': 'cfg5 S4→S1'}


def load(n):
    return json.load(open(os.path.join(ROOT, "profiles", f"r02_bench_default_n{n}.json")))["graph_switch"]


def replace_table(s, header, lines):
    start = s.index(header)
    end = s.index("\n\n", start)
    return s[:start] + "\n".join(lines) + s[end:]


def main():
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    gs = load(1)
    rec = {}
    for key in ("cold", "cfg5_cycle"):
        st = gs[key]["steps"]
        h = len(st) // 2
        for a, b in zip(st[:h], st[h:]):
            rec[a["step"]] = (a["plan_ms"], a["compile_ms"], a["first_run_ms"], a["total_ms"], b["warm_ms"])
    hdr = "| step | plan ms | compile ms | first run ms | cold ms | warm ms | cold / warm |"
    lines = [hdr, "|---|---|---|---|---|---|---|"]
    for k, v in NAMES.items():
        pl, co, fr, to, wa = rec[k]
        lines.append(f"| {v} | {pl:.2f} | {co:.2f} | {fr:.2f} | {to:.2f} | {wa:.2f} | {to / wa:.2f} |")
    lines.append(f"| cfg4 ↔ reverse cycle, pipelined | | | | {gs['cold']['pipelined']['cycle_ms']:.1f} "
                 f"| {gs['cold']['pipelined']['warm_cycle_ms']:.1f} | {gs['cold']['pipelined']['cold_over_warm']:.2f} |")
    lines.append(f"| cfg5 cycle, pipelined | | | | {gs['cfg5_cycle']['pipelined']['cycle_ms']:.1f} "
                 f"| {gs['cfg5_cycle']['pipelined']['warm_cycle_ms']:.1f} | {gs['cfg5_cycle']['pipelined']['cold_over_warm']:.2f} |")
    s = replace_table(s, hdr, lines)
    r = {n: load(n) for n in (2, 4)}

    def rows(g):
        out = {}
        for key in ("cold", "cfg5_cycle"):
            st = g[key]["steps"]
            for b in st[len(st) // 2:]:
                out[b["step"]] = (b["cold_total_ms"], b["warm_ms"], b["warm_tuned_ms"], b.get("tuned_flags"))
            out[key + "_pipe"] = g[key]["pipelined"]
        return out
    r2, r4 = rows(r[2]), rows(r[4])
    hdr = "| step | N=2 cold / warm / tuned (ms) | N=4 cold / warm / tuned (ms) |"
    lines = [hdr, "|---|---|---|"]
    for k, v in NAMES.items():
        a, b = r2[k], r4[k]
        lines.append(f"| {v} | {a[0]:.2f} / {a[1]:.2f} / {a[2]:.2f} (flags {a[3]}) | "
                     f"{b[0]:.2f} / {b[1]:.2f} / {b[2]:.2f} (flags {b[3]}) |")
    for key, label in (("cold_pipe", "cfg4 ↔ reverse cycle, pipelined cold / warm"),
                       ("cfg5_cycle_pipe", "cfg5 cycle, pipelined cold / warm")):
        a, b = r2[key], r4[key]
        lines.append(f"| {label} | {a['cycle_ms']:.1f} / {a['warm_cycle_ms']:.1f} ({a['cold_over_warm']:.2f}×) | "
                     f"{b['cycle_ms']:.1f} / {b['warm_cycle_ms']:.1f} ({b['cold_over_warm']:.2f}×) |")
    s = replace_table(s, hdr, lines)
    open(p, "w").write(s)


if __name__ == "__main__":
    main()
