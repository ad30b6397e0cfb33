"""Locate the reference package (``coserve``) this layer drops into.

The drop-in runs INSIDE the reference's control plane: its engine, dispatcher, coordinator and
launcher (/root/reference/pkg/src/coserve) stay unmodified and call this package at the replica
step.  When ``coserve`` is importable — installed in the environment, or in this repository's
git-ignored ``baseline/_ref`` (``pip install --target baseline/_ref <reference>/pkg``, the
driver's convention; it travels to the GPU box) — the package aliases the reference's own error
and value classes (``domain.ConfigurationError`` / ``InvariantViolation`` / ``Request`` /
``BatchConfig``, domain.py:15-98; ``launcher.AggregationError``, launcher.py:24-25), so an error
raised by the CUDA path is the very class the reference catches (experiment.py:43-48 maps
ConfigurationError to exit code 2).  Without the reference the package is self-contained.
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
_CANDIDATES = (ROOT / "baseline" / "_ref",)


def import_coserve(extra: tuple[str | Path, ...] = ()):
    """Return the ``coserve`` package, or None when it is not available."""
    try:
        return importlib.import_module("coserve")
    except ImportError:
        pass
    for p in (*map(Path, extra), *_CANDIDATES):
        if (p / "coserve" / "__init__.py").is_file():
            if str(p) not in sys.path:
                sys.path.append(str(p))
            try:
                return importlib.import_module("coserve")
            except ImportError:  # pragma: no cover - broken install
                continue
    return None


def coserve_module(name: str):
    """``coserve.<name>`` (e.g. 'engine', 'launcher'), or None without the reference."""
    pkg = import_coserve()
    if pkg is None:
        return None
    return importlib.import_module(f"coserve.{name}")
