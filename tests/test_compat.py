"""CPU: the remeshx drop-in switch rebinds every reindex name (needs the reference importable)."""
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present on this machine")
def test_install_into_remeshx_rebinds_all_names():
    sys.path.insert(0, REF)
    try:
        import remeshx
        import remeshx.ops
        import remeshx.pipeline
        import remeshx.bench  # noqa: F401
        import remeshx.cli  # noqa: F401
        import remeshx.testing  # noqa: F401
        from paper_2109_09812_b200.compat import install_into_remeshx
        saved = {m: sys.modules[m].reindex for m in ("remeshx", "remeshx.pipeline", "remeshx.ops",
                                                       "remeshx.bench", "remeshx.testing", "remeshx.cli")}
        try:
            patched = install_into_remeshx()
            assert set(patched) >= {"remeshx", "remeshx.pipeline", "remeshx.ops", "remeshx.bench",
                                    "remeshx.testing", "remeshx.cli"}
            fn = remeshx.reindex
            assert getattr(fn, "__wrapped_b200__", False)
            for m in patched:
                assert sys.modules[m].reindex is fn
        finally:
            for m, f in saved.items():
                sys.modules[m].reindex = f
    finally:
        sys.path.remove(REF)
