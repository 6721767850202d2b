import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(ROOT, "tests", "golden", "reference_vectors.npz")
    z = np.load(path)
    data = {k: z[k] for k in z.files}
    data["meta"] = json.loads(bytes(data.pop("meta_json")).decode())
    return data


@pytest.fixture(scope="session")
def oracle():
    from oracle import n2f_oracle

    return n2f_oracle
