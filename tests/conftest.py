import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device); run with -m gpu")
    config.addinivalue_line("markers", "exhaustive: whole-input-space oracle runs; set SINCOS_EXHAUSTIVE=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("SINCOS_EXHAUSTIVE") == "1":
        return
    skip = pytest.mark.skip(reason="whole-input-space run; set SINCOS_EXHAUSTIVE=1 "
                                   "(committed result: tests/golden/oracle_exhaustive.json)")
    for item in items:
        if "exhaustive" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(ROOT, "tests", "golden")
    out = {}
    for name in ("paper_values", "survey_crosscheck"):
        with open(os.path.join(d, name + ".json")) as f:
            out[name] = json.load(f)
    return out
