import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
CASES = ("heis6_p2", "hub4_p1", "ints4_p1", "ints6_d24_p2", "ints7_d32_p2")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(params=CASES)
def golden(request):
    from paper_2305_05581_b200.plan_input import PlanInput
    return request.param, PlanInput.load(os.path.join(GOLDEN, request.param + ".npz"))


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
