"""pytest plugin (test infrastructure): run the REFERENCE's own test suite
against the B200 drop-in.

The reference's tests import their entry points at collection time, so the
names are rebound before any test module is imported (three
names for conv_twostage — convkit.conv_twostage, convkit.twostage.conv_twostage,
convkit.bench.conv_twostage, /root/reference/pkg/src/convkit/__init__.py:18-20,
bench.py:25 — plus stage1_scalar_prods / stage2_sum, which TestStage1 /
TestStage2 call).  Each rebound function converts the reference's objects
(ConvConfig, Tensor4, DeviceModel, LaunchPlan, PartialSums) into the drop-in's,
calls the drop-in — which runs the paper-faithful two-stage engine on the GPU
through the C ABI — and converts results and exceptions back into the
reference's classes, so the tests' isinstance checks and pytest.raises hold.

    python -m pytest <convkit tests> -p reference_rebind   (tests/ on sys.path)
"""

from __future__ import annotations

import functools

import convkit
import convkit.bench as ck_bench
import convkit.twostage as ck_twostage

import paper_2103_16234_b200 as pk
import paper_2103_16234_b200.errors as pk_errors
from paper_2103_16234_b200 import twostage as ours

CALLS = {"conv_twostage": 0, "stage1_scalar_prods": 0, "stage2_sum": 0}


def _cfg(c):
    return pk.ConvConfig(c.name, n=c.n, c=c.c, h=c.h, w=c.w, m=c.m, hf=c.hf, wf=c.wf, stride=c.stride,
                         pad_h=c.pad_h, pad_w=c.pad_w)


def _t4(t):
    return pk.Tensor4(t.data) if t is not None and hasattr(t, "data") else t


def _dev(d):
    if d is None:
        return None
    return pk.DeviceModel(warp_width=d.warp_width, line_bytes=d.line_bytes,
                          max_threads_per_block=d.max_threads_per_block, element_bytes=d.element_bytes)


def _plan(p):
    if p is None:
        return None
    return pk.LaunchPlan(blocks=p.blocks, threads_per_block=p.threads_per_block,
                         split_per_filter_row=p.split_per_filter_row,
                         dot_products_per_thread=p.dot_products_per_thread)


def _stats(s):
    return ck_twostage.RunStats(stage1_tasks_run=s.stage1_tasks_run, stage2_invoked=s.stage2_invoked,
                                filter_row_global_loads=s.filter_row_global_loads,
                                workspace_bytes=s.workspace_bytes)


def _reraise(exc):
    """The drop-in's exception -> the reference class of the same name."""
    if isinstance(exc, pk_errors.WorkspaceExceeded):
        return convkit.WorkspaceExceeded(exc.required, exc.limit)
    if isinstance(exc, pk_errors.InvalidConfig):
        return convkit.InvalidConfig(exc.field, str(exc).split(": ", 1)[-1])
    cls = getattr(convkit, type(exc).__name__, None)
    if cls is not None and isinstance(exc, pk_errors.ConvKitError):
        return cls(str(exc))
    return exc


def _translated(name):
    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*a, **k):
            CALLS[name] += 1
            try:
                return fn(*a, **k)
            except pk_errors.ConvKitError as exc:
                raise _reraise(exc) from exc
        return wrapper
    return deco


@_translated("conv_twostage")
def conv_twostage(inp, filters, cfg, device=None, workspace_limit=ck_twostage.DEFAULT_WORKSPACE_LIMIT, *,
                  plan=None, workers=1):
    out, stats = ours.conv_twostage(_t4(inp), _t4(filters), _cfg(cfg), _dev(device), workspace_limit,
                                    plan=_plan(plan), workers=workers)
    return convkit.Tensor4(out.data), _stats(stats)


@_translated("stage1_scalar_prods")
def stage1_scalar_prods(inp, filters, cfg, plan=None, *, device=None,
                        workspace_limit=ck_twostage.DEFAULT_WORKSPACE_LIMIT, workers=1):
    partials, stats = ours.stage1_scalar_prods(_t4(inp), _t4(filters), _cfg(cfg), _plan(plan), device=_dev(device),
                                               workspace_limit=workspace_limit, workers=workers)
    return ck_twostage.PartialSums(partials.data), _stats(stats)


@_translated("stage2_sum")
def stage2_sum(partials, cfg, *, workers=1):
    out, stats = ours.stage2_sum(ours.PartialSums(partials.data), _cfg(cfg), workers=workers)
    return convkit.Tensor4(out.data), _stats(stats)


for mod in (convkit, ck_twostage, ck_bench):
    for fname, fn in (("conv_twostage", conv_twostage), ("stage1_scalar_prods", stage1_scalar_prods),
                      ("stage2_sum", stage2_sum)):
        if hasattr(mod, fname):
            setattr(mod, fname, fn)


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"reference_rebind: drop-in calls {CALLS}")
