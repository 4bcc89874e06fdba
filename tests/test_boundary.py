"""The drop-in boundary: the C ABI and the reference-compatible C++ API.

* libhshard_b200.so loads and exports every entry point include/hshard_c.h
  declares, and the reference C++ API symbols (hshard::classify, fuse, ...).
* tests/cpp/api_test (compiled against include/hshard/*.hpp exactly as a
  reference user would) passes its planner / Tensor / scatter / reassemble
  checks on CPU, and execute_plan / apply_switch checks on the GPU.
* Errors cross the C ABI as 1 + Errc with the reference's Errc names.
"""
import os
import re
import subprocess
import sys

import pytest

from paper_2504_20490_b200 import LIB_PATH, hshard as H
from paper_2504_20490_b200._lib import ERRC_NAMES, LIB

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
API_TEST = os.path.join(ROOT, "tests", "cpp", "api_test")


def _declared():
    src = open(os.path.join(ROOT, "include", "hshard_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z_0-9]+)\s*\(", src)))


def test_c_abi_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(LIB, n)]
    assert not missing, missing


def test_cpp_api_symbols_exported():
    out = subprocess.run(["nm", "-DC", LIB_PATH], capture_output=True, text=True).stdout
    for sym in ["hshard::classify(", "hshard::build_table(", "hshard::fuse(", "hshard::make_plan(",
                "hshard::placement(", "hshard::convert_hsize(", "hshard::bottom_resolve(",
                "hshard::top_resolve(", "hshard::execute_plan(", "hshard::apply_switch(",
                "hshard::plan_switch(", "hshard::reassemble(", "hshard::scatter(",
                "hshard::volume_report(", "hshard::Tensor::slice(", "hshard::deduce_graph(",
                "hshard::CompGraph::dot(", "hshard::unify_inputs(", "hshard::diff_strategies(hshard::CompGraph",
                "hshard::instantiate(", "hshard::construct_pipelines(", "hshard::assign_schedule("]:
        assert sym in out, sym


def test_errc_names_match_reference_order():
    # reference common.hpp:34-70 order, executor codes appended
    assert ERRC_NAMES[:26][-1] == "ParseError"
    for i, name in enumerate(ERRC_NAMES):
        assert LIB.hs_errc_name(i).decode() == name
    with pytest.raises(H.HshardError) as ei:
        H.classify("hsize=1 hdim=-1 [(0,1,2,3){-2:4}]", "hsize=1 hdim=-1 [(0,1){0:2}]", [8, 8])
    assert ei.value.code == "PartialUnderBsr"
    with pytest.raises(H.HshardError) as ei:
        H.classify("not an annotation", "hsize=1 hdim=-1 [(0){}]", [8])
    assert ei.value.code == "ParseError"


def test_cpp_api_cpu():
    res = subprocess.run([API_TEST, "cpu"], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr


@pytest.mark.gpu
def test_cpp_api_gpu():
    res = subprocess.run([API_TEST, "gpu"], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr


def test_library_does_not_pin_nccl_before_torch():
    """libhshard_b200.so must not link libnccl: loaded before torch it would bind
    libnccl.so.2 to the system NCCL and break torch's own NCCL symbols."""
    out = subprocess.run(["ldd", LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl" not in out
    res = subprocess.run([sys.executable, "-c",
                          "import paper_2504_20490_b200, torch, torch.distributed; print('ok')"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]
