"""Drop-in switch for callers of the reference package `jetpart`.

`install()` loads the reference package (from `baseline/_ref`, or any path
holding a `jetpart/` directory) under a private name and rebinds every
hot-path entry point in each of its modules to this package's GPU
implementation, then registers the patched modules as `jetpart` and
`jetpart.<module>` in `sys.modules`. The reference's host-side code (METIS /
MatrixMarket I/O, the CLI, the scikit-learn estimator, the generators,
`preprocess`, the rebalancing scalar helpers) keeps running unchanged, but
every call it makes into the partitioner lands on the GPU path. This is the
binding a maintainer adds to switch.

Rebound names (reference file:line -> here):
  driver.py:24-126      partition, project, PartitionResult
  coarsen.py:19-161     Hierarchy, match_vertices, contract, build_hierarchy
  refine.py:78-294      select_destinations, afterburner, jetlp_pass, jet_refine
  rebalance.py:139-240  weak_rebalance_pass, strong_rebalance_pass
  conn.py:29-272        ConnectivityTable, build_conn, update_conn
  initpart.py:70-94     initial_partition
  graph.py:215-221      cutsize
  moves.py:12-39        MoveList
  errors.py:4-33        the exception classes (so `except` clauses match)

Mode: the reference has one (deterministic) behaviour; `partition` runs in
this package's deterministic mode (bit-identical results) unless
JETPART_COMPAT_MODE=throughput is set, which selects the throughput mode
(hashed-priority matching; cut within 2 % of the reference, balance met).
"""

from __future__ import annotations

import dataclasses
import importlib
import importlib.util
import os
import sys
from pathlib import Path

from . import driver as _driver
from . import errors as _errors
from . import graph as _graph
from . import moves as _moves
from . import ops as _ops

_PRIVATE = "_jetpart_reference"
_MODULES = ("errors", "_arrays", "_validation", "graph", "moves", "conn", "coarsen", "initpart",
            "refine", "rebalance", "driver", "io", "generators", "estimator", "cli")


def _mode_config(config):
    det = os.environ.get("JETPART_COMPAT_MODE", "deterministic") != "throughput"
    if dataclasses.is_dataclass(config) and hasattr(config, "deterministic"):
        return dataclasses.replace(config, deterministic=det)
    config.deterministic = det
    return config


def partition(graph, config):
    """jetpart.driver.partition on the GPU (driver.py:48-126)."""
    return _driver.partition(graph, _mode_config(config))


def jet_refine(graph, state, config, finest=True, seed_path=()):
    """jetpart.refine.jet_refine on the GPU (refine.py:190-294)."""
    return _ops.jet_refine(graph, state, config, finest=finest, seed_path=seed_path)


def overrides() -> dict:
    return {
        "partition": partition,
        "project": _driver.project,
        "PartitionResult": _driver.PartitionResult,
        "Hierarchy": _ops.Hierarchy,
        "match_vertices": _ops.match_vertices,
        "contract": _ops.contract,
        "build_hierarchy": _ops.build_hierarchy,
        "select_destinations": _ops.select_destinations,
        "afterburner": _ops.afterburner,
        "jetlp_pass": _ops.jetlp_pass,
        "jet_refine": jet_refine,
        "weak_rebalance_pass": _ops.weak_rebalance_pass,
        "strong_rebalance_pass": _ops.strong_rebalance_pass,
        "ConnectivityTable": _ops.ConnectivityTable,
        "build_conn": _ops.build_conn,
        "update_conn": _ops.update_conn,
        "initial_partition": _ops.initial_partition,
        "cutsize": _graph.cutsize,
        "MoveList": _moves.MoveList,
        "JetpartError": _errors.JetpartError,
        "ParseError": _errors.ParseError,
        "PreprocessError": _errors.PreprocessError,
        "BalanceInfeasibleError": _errors.BalanceInfeasibleError,
        "RebalanceInfeasibleError": _errors.RebalanceInfeasibleError,
    }


def _default_root() -> Path:
    env = os.environ.get("JETPART_REFERENCE")
    if env:
        return Path(env)
    return Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def install(root=None):
    """Load the reference from `root` (a directory containing `jetpart/`),
    rebind its hot path to this package and register it as `jetpart`.
    Returns the patched top-level module. Idempotent."""
    if "jetpart" in sys.modules and getattr(sys.modules["jetpart"], "_jet_b200_compat", False):
        return sys.modules["jetpart"]
    pkg_dir = Path(root or _default_root()) / "jetpart"
    if not (pkg_dir / "__init__.py").exists():
        raise ImportError(f"reference package not found at {pkg_dir}")
    # import the reference's submodules under a private package name, then
    # patch each module's namespace (functions defined there look names up in
    # their own module globals, so e.g. the estimator's fit() calls our
    # partition)
    spec = importlib.util.spec_from_file_location(
        _PRIVATE, pkg_dir / "__init__.py", submodule_search_locations=[str(pkg_dir)])
    top = importlib.util.module_from_spec(spec)
    sys.modules[_PRIVATE] = top
    subs = {}
    for name in _MODULES:
        if (pkg_dir / f"{name}.py").exists():
            subs[name] = importlib.import_module(f"{_PRIVATE}.{name}")
    spec.loader.exec_module(top)
    ov = overrides()
    for mod in list(subs.values()) + [top]:
        for key, val in ov.items():
            if key in vars(mod):
                setattr(mod, key, val)
    top._jet_b200_compat = True
    sys.modules["jetpart"] = top
    for name, mod in subs.items():
        # leaf entry modules (`python -m jetpart.cli`) are left to the import
        # system: a fresh jetpart.cli binds the patched names of its parent
        if name != "cli":
            sys.modules[f"jetpart.{name}"] = mod
    return top
