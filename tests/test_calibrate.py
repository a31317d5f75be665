"""Native offline calibration (pasa_calibrate, host code in libpasa.so; SURVEY.md
§8f NEXT 2) against the oracle (Eqs. 9-11): same arithmetic in the same order,
so the tables are compared bit for bit.  No GPU work is involved."""
import numpy as np
import pytest

import oracle
from paper_2604_12219_b200 import _C
from paper_2604_12219_b200 import calibrate as C


@pytest.mark.parametrize("seed,N,rho", [(0, 1, 0.15), (1, 5, 0.15), (2, 10, 0.5), (3, 3, 0.05)])
def test_native_table_equals_oracle_bitwise(seed, N, rho):
    rng = np.random.default_rng(seed)
    curves = rng.uniform(0.1, 2.0, (N, 50))
    curves[:, :10] = np.nan                    # dense steps: ignored
    curves[0, 20] = 30.0                       # a clipped step at rho >= 0.15
    a = C.calibrate(curves, rho=rho)
    b = oracle.calibrate(curves, rho=rho)
    assert a["l1_mean"] == b["l1_mean"]
    assert np.array_equal(a["rho_table"], b["rho_table"])
    assert np.array_equal(a["alpha"], b["alpha"])
    assert np.array_equal(a["clipped"], b["clipped"])


def test_native_errors():
    with pytest.raises(_C.PasaError) as e:
        C.calibrate(np.zeros((2, 50)))
    assert e.value.status == _C.PASA_EDEGENERATE
    bad = np.ones((1, 50))
    bad[0, 30] = np.inf
    with pytest.raises(_C.PasaError) as e:
        C.calibrate(bad)
    assert e.value.status == _C.PASA_EINVAL
    with pytest.raises(_C.PasaError):
        C.calibrate(np.ones((1, 3)), dense_frac=1.0)
