import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    import oracles
    r = oracles.ref()
    if r is None:
        pytest.skip("oracle/_ref/libgss_ref.so not built (needs /root/reference at build time)")
    return r


@pytest.fixture(scope="session")
def orc():
    import oracles
    o = oracles.orc()
    if o is None:
        pytest.skip("oracle/_ref/libgss_oracle.so not built (make -C oracle oracle)")
    return o


@pytest.fixture(scope="session")
def parity_log():
    """Records measured deviations per test (max rel_err / rel_err_floor / abs) into the JSON file
    named by GSS_PARITY_OUT (default gpurun_out/parity.json when that directory exists), so the
    numbers behind the tolerances are committed (profiles/parity_r02.json), not just the dots."""
    import json
    import os

    path = os.environ.get("GSS_PARITY_OUT")
    if path is None and (ROOT / "gpurun_out").is_dir():
        path = str(ROOT / "gpurun_out" / "parity.json")
    rec = {}

    def log(name, **kv):
        rec[name] = {k: (float(v) if hasattr(v, "__float__") and not isinstance(v, (int, bool)) else v)
                     for k, v in kv.items()}
        if path:
            old = {}
            try:
                with open(path) as f:
                    old = json.load(f)
            except Exception:
                pass
            old.update(rec)
            with open(path, "w") as f:
                json.dump(old, f, indent=1, sort_keys=True)

    return log
