import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="module")
def gpu_ctx():
    """One executor context on cuda:0 per test module (closed before the
    multi-GPU tests, whose rank 0 needs that memory on the same GPU)."""
    if not cuda_available():
        pytest.skip("no GPU")
    import torch
    from paper_2504_20490_b200 import executor
    free, total = torch.cuda.mem_get_info(0)
    gb = int(os.environ.get("HS_TEST_ARENA_GB", "0")) or max(4, int(free / 2**30) - 12)
    ctx = executor.Context(arena_bytes=gb << 30)
    yield ctx
    ctx.close()
