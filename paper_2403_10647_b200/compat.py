"""Injection shim: make a live reference `pargrid` import use the B200 builder.

    import pargrid
    from paper_2403_10647_b200 import compat
    compat.install(pargrid)        # before `from pargrid import build_parallel` elsewhere

replaces, in place (SURVEY.md §8b "Callers"):
  * pargrid.builders.build_parallel and pargrid.build_parallel  (builders.py:144)
  * pargrid.builders.build_sorted / build_compact (+ pargrid.*) (builders.py:172, 195)
    -- the GPU comparison builders of SURVEY §8(f) row 1 (algos="all")
  * pargrid.cli.ALGORITHMS[...] for each replaced builder       (cli.py:30-34)
  * pargrid.stats.compute_stats and pargrid.compute_stats       (stats.py:43; GPU reductions,
    with consumers=True)
  * pargrid.geometry.load_obj (+ its re-exports)                (geometry.py:84; GPU parser,
    with consumers=True)
  * pargrid.kernels._BACKENDS["cuda"]                           (kernels/__init__.py:17-19)
    -- radix_sort_pairs and dda_cast on the GPU
The wrapper returns the reference's own CompactGrid / BuildReport types, raises the
reference's own error classes and honours pargrid.builders._fault_inject, so the
reference's test-suite runs unchanged against the GPU path (tests/test_reference_suite.py).
"""

import sys
import types

from . import builders as _b
from . import errors as _e
from . import kernels as _k
from . import obj as _o
from . import stats as _s


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


def _make_builder(pargrid, ours, has_record, fault_hook):
    perr = pargrid.errors
    pbuilders = sys.modules["pargrid.builders"]
    pgridcore = sys.modules["pargrid.gridcore"]

    def convert(spec, grid, rep):
        O = grid.O
        if fault_hook and pbuilders._fault_inject and rep.no:
            O = O.copy()
            O[0] ^= 1
        report = pbuilders.BuildReport(rep.algo, no=rep.no, max_task_work=rep.max_task_work,
                                       total_work=rep.total_work, phase_ms=dict(rep.phase_ms))
        return pgridcore.CompactGrid(spec, grid.G, O), report

    if has_record:
        def build(mesh, spec, workers=None, record=None):
            return convert(spec, *_wrap_errors(ours, perr)(mesh, spec, workers=workers, record=record))
    else:
        def build(mesh, spec, workers=None):
            return convert(spec, *_wrap_errors(ours, perr)(mesh, spec, workers=workers))
    build.__name__ = ours.__name__
    build.__doc__ = ours.__doc__
    build.__wrapped_b200__ = True
    return build


def make_build_parallel(pargrid):
    return _make_builder(pargrid, _b.build_parallel, True, True)


def make_build_sorted(pargrid):
    return _make_builder(pargrid, _b.build_sorted, True, True)


def make_build_compact(pargrid):
    return _make_builder(pargrid, _b.build_compact, False, False)


def make_compute_stats(pargrid):
    perr = pargrid.errors
    pstats = sys.modules["pargrid.stats"]

    def compute_stats(grid, mesh):
        st = _wrap_errors(_s.compute_stats, perr)(grid, mesh)
        return pstats.GridStats(**{f: getattr(st, f) for f in st.__dataclass_fields__})

    compute_stats.__doc__ = _s.compute_stats.__doc__
    compute_stats.__wrapped_b200__ = True
    return compute_stats


def make_load_obj(pargrid):
    perr = pargrid.errors
    pgeom = sys.modules["pargrid.geometry"]

    def load_obj(path):
        try:
            mesh = _o.load_obj(path)
        except _e.ObjParseError as exc:
            msg = str(exc)
            prefix = f"line {exc.line_number}: "
            raise perr.ObjParseError(msg[len(prefix):] if msg.startswith(prefix) else msg,
                                     exc.line_number) from exc
        return pgeom.TriangleMesh(mesh.vertices, mesh.triangles)

    load_obj.__doc__ = _o.load_obj.__doc__
    load_obj.__wrapped_b200__ = True
    return load_obj


def make_backend(pargrid):
    kernels = sys.modules["pargrid.kernels"]
    lane = kernels._BACKENDS.get("c") or kernels._BACKENDS["python"]
    mod = types.ModuleType("pargrid_cuda_lane")
    mod.BACKEND_NAME = _k.BACKEND_NAME
    mod.radix_sort_pairs = _k.radix_sort_pairs
    mod.dda_cast = _k.dda_cast
    for name in ("pairgen_sorted", "compact_count", "compact_fill"):
        setattr(mod, name, getattr(lane, name))
    return mod


def install(pargrid=None, backend=True, algos=("parallel",), consumers=False):
    """algos: which builders to replace ("parallel", "sorted", "compact", or "all");
    consumers: also replace compute_stats (ray casting goes through the "cuda" lane)."""
    if pargrid is None:
        import pargrid  # noqa: F401
        pargrid = sys.modules["pargrid"]
    if algos == "all":
        algos = ("parallel", "sorted", "compact")
    makers = {"parallel": make_build_parallel, "sorted": make_build_sorted, "compact": make_build_compact}
    cli = sys.modules.get("pargrid.cli")
    if cli is None:
        import importlib
        cli = importlib.import_module("pargrid.cli")
    bp = None
    for algo in algos:
        fn = makers[algo](pargrid)
        setattr(sys.modules["pargrid.builders"], f"build_{algo}", fn)
        setattr(pargrid, f"build_{algo}", fn)
        cli.ALGORITHMS[algo] = fn
        if algo == "parallel":
            bp = fn
    if consumers:
        import importlib
        pstats = importlib.import_module("pargrid.stats")
        cs = make_compute_stats(pargrid)
        pstats.compute_stats = cs
        pargrid.compute_stats = cs
        cli.compute_stats = cs
        lo = make_load_obj(pargrid)
        sys.modules["pargrid.geometry"].load_obj = lo
        for mod in (pargrid, cli):
            if hasattr(mod, "load_obj"):
                mod.load_obj = lo
    if backend:
        sys.modules["pargrid.kernels"]._BACKENDS["cuda"] = make_backend(pargrid)
    return bp
