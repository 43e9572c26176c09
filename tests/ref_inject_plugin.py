"""pytest plugin: inject the B200 builder into the reference package before its test-suite
collects (used by tests/test_reference_suite.py)."""


def pytest_configure(config):
    import pargrid

    from paper_2403_10647_b200 import compat
    compat.install(pargrid)
