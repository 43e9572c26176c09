"""pytest plugin: inject the B200 builders into the reference package before its test-suite
collects (used by tests/test_reference_suite.py). PGRID_INJECT_ALGOS="all" also replaces
build_sorted / build_compact with the GPU comparison builders."""

import os


def pytest_configure(config):
    import pargrid

    from paper_2403_10647_b200 import compat
    algos = os.environ.get("PGRID_INJECT_ALGOS", "parallel")
    compat.install(pargrid, algos="all" if algos == "all" else tuple(algos.split(",")),
                   consumers=algos == "all")
