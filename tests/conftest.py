import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(autouse=True, scope="module")
def _release_gpu_scratch():
    """GPU test modules may leave a large shared generation workspace (half the
    free device memory at C5); release it between modules."""
    yield
    import sys as _sys
    gen = _sys.modules.get("paper_2206_08660_b200.generate")
    if gen is not None:
        gen.release_workspace()
        torch = _sys.modules.get("torch")
        if torch is not None and torch.cuda.is_available():
            torch.cuda.empty_cache()
