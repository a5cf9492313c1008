"""pytest plugin: run the reference remeshx test-suite against the B200 path.

    PYTHONPATH=<remeshx src>:<this repo>:<this repo>/integration \
        pytest -p remeshx_b200_plugin <remeshx>/tests

Loaded with -p it runs before the test modules import ``reindex`` by name
(SURVEY.md section 4.3), so every binding sees the B200 implementation.  The
header names the patched bindings and the loaded CUDA library; the terminal
summary counts the calls that went through it.
"""

_STATE = {"patched": [], "calls": 0}


def pytest_configure(config):
    from paper_2109_09812_b200 import compat
    _STATE["patched"] = compat.install_into_remeshx(on_call=_count)


def _count():
    _STATE["calls"] += 1


def pytest_report_header(config):
    from paper_2109_09812_b200 import _native
    lib = _native.lib()
    return [f"remeshx_b200: reindex rebound in {', '.join(_STATE['patched'])}",
            f"remeshx_b200: CUDA library {_native.LIB_PATH} ({lib.rmx_version().decode()})"]


def pytest_terminal_summary(terminalreporter):
    from paper_2109_09812_b200 import _native
    terminalreporter.write_line(
        f"remeshx_b200: {_STATE['calls']} reindex calls ran on the B200 path "
        f"({_native.lib().rmx_kernel_launches_total()} kernel launches)")
