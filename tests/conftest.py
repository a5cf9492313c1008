import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
GROUPS = ("worked", "reftests", "torture", "random", "grid", "lattice")
FIELDS = ("is_used", "org_id", "nodup", "new_idx", "perm")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: full-size configs")


def load_group(group: str) -> dict:
    """{case name: {field: array}} of one golden fixture file (made by tools/make_golden.py
    from the reference remeshx.reindex)."""
    data = np.load(os.path.join(GOLDEN, f"{group}.npz"))
    cases: dict = {}
    for key in data.files:
        name, field = key.rsplit("/", 1)
        cases.setdefault(name, {})[field] = data[key]
    return cases


def all_golden() -> list[tuple[str, dict]]:
    out = []
    for g in GROUPS:
        for name, case in sorted(load_group(g).items()):
            out.append((f"{g}:{name}", case))
    return out


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def pytest_sessionfinish(session, exitstatus):
    """With the bounds-counting build loaded (RMX_LIB=.../librmx_b200_checked.so), report the
    scattered stores whose index was past its array over the whole session, and fail on any."""
    import ctypes
    if "paper_2109_09812_b200._native" not in sys.modules:
        return
    native = sys.modules["paper_2109_09812_b200._native"]
    if native._lib is None:
        return
    oob = ctypes.c_ulonglong(0)
    try:
        rc = native._lib.rmx_debug_oob_count(ctypes.byref(oob))
    except Exception:  # noqa: BLE001 - no device / not loaded
        return
    if rc == 0:
        print(f"\nchecked build: {oob.value} out-of-bounds scattered stores in this session")
        if oob.value:
            session.exitstatus = 1
