"""pytest plugin: run the reference remeshx test-suite against the B200 path.

    PYTHONPATH=<remeshx src>:<this repo>:<this repo>/integration \
        pytest -p remeshx_b200_plugin <remeshx>/tests

Loaded with -p it runs before the test modules import ``reindex`` by name
(SURVEY.md section 4.3), so every binding sees the B200 implementation.
"""


def pytest_configure(config):
    from paper_2109_09812_b200.compat import install_into_remeshx
    patched = install_into_remeshx()
    config.stash_b200_patched = patched  # for -v reporting / debugging
