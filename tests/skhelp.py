"""Shared helpers for the test-suite (golden fixtures, GPU guards)."""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def import_soakit():
    """The reference package as test infrastructure: the gitignored install
    under baseline/_ref (travels to the GPU box), else the read-only source
    tree in the dev container. None when neither exists."""
    import importlib
    import sys

    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "soakit")):
            if path not in sys.path:
                sys.path.append(path)
            return importlib.import_module("soakit")
    return None
