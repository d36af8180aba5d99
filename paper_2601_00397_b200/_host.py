"""Exception bridging to the host framework (the reference package ``timewarp``).

When ``timewarp`` is importable, this engine's drop-in exception classes also derive
from the host's classes of the same name, so host code written against the reference
(``except timewarp.predictor.TableMiss``, ``except timewarp.oracle.OracleStalled``)
catches them unchanged. Without the host the classes stand alone."""

from __future__ import annotations

import importlib


def host_bases(module: str, name: str) -> tuple:
    """(timewarp.<module>.<name>,) if importable and an Exception class, else ()."""
    try:
        mod = importlib.import_module(f"timewarp.{module}")
    except Exception:
        return ()
    cls = getattr(mod, name, None)
    return (cls,) if isinstance(cls, type) and issubclass(cls, Exception) else ()


def host_module(module: str):
    """timewarp.<module> when the host framework is importable, else None."""
    try:
        return importlib.import_module(f"timewarp.{module}")
    except Exception:
        return None
