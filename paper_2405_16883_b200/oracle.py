"""Counterpart of the reference's ``sparsetc.oracle`` module (`/root/reference/pkg/src/sparsetc/oracle.py:19-46`,
re-exported by `__init__.py:27`): ``eval_dense``, the brute-force dense evaluation of an
expression (float64, ascending reduction; implemented in ``dense_eval``), so that
``from paper_2405_16883_b200.oracle import eval_dense`` works like ``from sparsetc.oracle import eval_dense``.

This is the reference's public API, not the parity oracle of the test suite (the repo-root
``oracle/`` package), which nothing in this package imports.
"""

from .dense_eval import eval_dense

__all__ = ["eval_dense"]
