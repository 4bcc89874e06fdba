"""NCCL-convention bus bytes against the figures SURVEY
§8(d)'s table quotes from the compiled reference planner."""
from paper_2504_20490_b200 import hshard as H
from paper_2504_20490_b200 import workloads as W
from paper_2504_20490_b200.accounting import bus_bytes

MiB = 1 << 20


def _plan(name):
    w = W.by_name(name)
    if w.kind == "classify":
        t, s, d, sh = w.transitions[0]
        return H.classify(s, d, sh, w.dtype)
    return H.plan_switch(w.transitions, w.dtype)


def test_cfg2e_bus_bytes():
    b = bus_bytes(_plan("cfg2e"))
    # RS4 of a 128 MiB partial box = 96 MiB; RS2 = 64 MiB; SplitRS pieces 16 / 32 MiB
    assert b[0] == 96 * MiB + 16 * MiB
    assert max(b.values()) == 160 * MiB  # SURVEY: max per GPU per direction 160 MiB


def test_cfg3a_naive_split_allreduce_fanout():
    b = bus_bytes(_plan("cfg3a"))
    # AR4 of 1 GiB = 1.5 GiB, plus the lowest-id contributor's 7 GiB fan-out
    assert b[0] == b[4] == 1536 * MiB + 7 * 1024 * MiB
    assert b[1] == 1536 * MiB


def test_cfg4_switch_sender_bytes():
    b = bus_bytes(_plan("cfg4"))
    assert sum(b.values()) == sum(x[4] for x in _plan("cfg4").json()["xfer"])
    assert abs(sum(b.values()) / 1e9 - 10.108) < 0.001  # SURVEY: 10.108 GB of transfers
    assert abs(max(b.values()) / 1e9 - 1.750) < 0.001   # max send 1.750 GB (GPU 1 / 6)


def test_cfg1b_bsr_transfers():
    b = bus_bytes(_plan("cfg1B"))
    assert sum(b.values()) == 134217728  # SURVEY: 2x50.3 MB + 2x16.8 MB
