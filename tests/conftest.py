import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def load_golden(name):
    import numpy as np
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden


# Observed parity errors (max over the checked rows/heads), written to $BSFA_PARITY_METRICS at the end
# of the session so the margins behind ROW_RTOL / LSE_ATOL / ATOL can be committed under profiles/.
PARITY_METRICS = {}


def record_metric(name, value):
    PARITY_METRICS[name] = max(float(value), PARITY_METRICS.get(name, float("-inf")))


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("BSFA_PARITY_METRICS")
    if path and PARITY_METRICS:
        import json
        with open(path, "w") as f:
            json.dump(PARITY_METRICS, f, indent=1, sort_keys=True)
