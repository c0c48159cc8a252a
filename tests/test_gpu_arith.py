"""The exact arithmetic shortcuts, checked on the device itself
(vdi_selftest_arith): Markstein division == IEEE division, __drcp_rn(n) ==
1.0 / n, d2 >= thr(g) <=> sqrt(d2) >= g (including d2 within a few ulps of
thr), and the shared-reciprocal transform == three IEEE divisions."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2206_08660_b200 import _capi  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402


def test_exact_shortcuts_have_no_mismatch():
    bad = torch.zeros(4, dtype=torch.int64, device="cuda")
    for seed in (1, 2, 3):
        _capi.check(_capi.load().vdi_selftest_arith(20_000_000, seed, dv.ptr(bad),
                                                    dv.stream_handle()))
        counts = dv.to_host(bad)
        assert np.all(counts == 0), counts
