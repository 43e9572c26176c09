"""Injection shim: make a live reference `pargrid` import use the B200 builder.

    import pargrid
    from paper_2403_10647_b200 import compat
    compat.install(pargrid)        # before `from pargrid import build_parallel` elsewhere

replaces, in place (SURVEY.md §8b "Callers"):
  * pargrid.builders.build_parallel and pargrid.build_parallel  (builders.py:144)
  * pargrid.cli.ALGORITHMS["parallel"]                          (cli.py:30-34)
  * pargrid.kernels._BACKENDS["cuda"]                           (kernels/__init__.py:17-19)
The wrapper returns the reference's own CompactGrid / BuildReport types, raises the
reference's own error classes and honours pargrid.builders._fault_inject, so the
reference's test-suite runs unchanged against the GPU path (tests/test_reference_suite.py).
"""

import sys
import types

from . import builders as _b
from . import errors as _e
from . import kernels as _k


def _wrap_errors(fn, perr):
    mapping = ((_e.SizeError, perr.SizeError), (_e.InvariantError, perr.InvariantError),
               (_e.ObjParseError, perr.ObjParseError), (_e.GridError, perr.GridError))

    def call(*a, **kw):
        try:
            return fn(*a, **kw)
        except _e.GridError as exc:
            for ours, theirs in mapping:
                if isinstance(exc, ours):
                    raise theirs(str(exc)) from exc
            raise
    return call


def make_build_parallel(pargrid):
    perr = pargrid.errors
    pbuilders = sys.modules["pargrid.builders"]
    pgridcore = sys.modules["pargrid.gridcore"]

    def build_parallel(mesh, spec, workers=None, record=None):
        grid, rep = _wrap_errors(_b.build_parallel, perr)(mesh, spec, workers=workers, record=record)
        O = grid.O
        if pbuilders._fault_inject and rep.no:
            O = O.copy()
            O[0] ^= 1
        report = pbuilders.BuildReport(rep.algo, no=rep.no, max_task_work=rep.max_task_work,
                                       total_work=rep.total_work, phase_ms=dict(rep.phase_ms))
        return pgridcore.CompactGrid(spec, grid.G, O), report

    build_parallel.__doc__ = _b.build_parallel.__doc__
    build_parallel.__wrapped_b200__ = True
    return build_parallel


def make_backend(pargrid):
    kernels = sys.modules["pargrid.kernels"]
    lane = kernels._BACKENDS.get("c") or kernels._BACKENDS["python"]
    mod = types.ModuleType("pargrid_cuda_lane")
    mod.BACKEND_NAME = _k.BACKEND_NAME
    mod.radix_sort_pairs = _k.radix_sort_pairs
    for name in ("pairgen_sorted", "compact_count", "compact_fill", "dda_cast"):
        setattr(mod, name, getattr(lane, name))
    return mod


def install(pargrid=None, backend=True):
    if pargrid is None:
        import pargrid  # noqa: F401
        pargrid = sys.modules["pargrid"]
    bp = make_build_parallel(pargrid)
    sys.modules["pargrid.builders"].build_parallel = bp
    pargrid.build_parallel = bp
    cli = sys.modules.get("pargrid.cli")
    if cli is None:
        import importlib
        cli = importlib.import_module("pargrid.cli")
    cli.ALGORITHMS["parallel"] = bp
    if backend:
        sys.modules["pargrid.kernels"]._BACKENDS["cuda"] = make_backend(pargrid)
    return bp
