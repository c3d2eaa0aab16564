"""Seeded synthetic workloads (graphs, S sets, initial states) for MulMent.

Shared by the oracle tests, the GPU tests and bench.py; holds none of the
method's arithmetic (see DESIGN.md §"Input recipe")."""
from . import configs, graphs, sset  # noqa: F401
