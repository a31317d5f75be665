import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


# ---- achieved-error log of the GPU parity tests (record every case) ----
_ERRORS = []


@pytest.fixture
def parity_log(request):
    """Append one achieved-error record per compared output: the test id, the
    case label, max|O_gpu - O_ref| / max|O_ref| and the relative Frobenius error.
    Written at session end to $PASA_PARITY_LOG (default gpurun_out/parity_errors.json)
    when any record exists; tools/parity_table.py turns it into profiles/ markdown."""
    def log(label, max_rel, frob_rel, bound, ref="oracle"):
        _ERRORS.append(dict(test=request.node.nodeid, case=label, max_rel=float(max_rel),
                            frob_rel=float(frob_rel), bound=float(bound), ref=ref))
    return log


def pytest_sessionfinish(session, exitstatus):
    if not _ERRORS:
        return
    import json
    path = os.environ.get("PASA_PARITY_LOG", os.path.join(ROOT, "gpurun_out",
                                                          "parity_errors.json"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(_ERRORS, f, indent=1)
