"""A bounded slice of the randomised parity fuzzer (tools/fuzz_parity.py) in
the GPU suite: 400 random cases (family x dtype x shape x alignment x input
mode x k-bit table) against the float64 oracle with the DESIGN 7 bars.  The
long runs (tens of thousands of cases) are in profiles/r02/session4/."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_fuzz_slice(seed):
    import fuzz_parity
    fails = fuzz_parity.run_cases(seed, 100)
    assert not fails, fails[:5]
