"""Seeded synthetic inputs and workload shapes shared by tests, bench and oracle.

This module deliberately holds NONE of the KS method's arithmetic: it only
draws random numbers and lists the pattern tuples / batch sizes of the
workloads. Both the CUDA path (through tests and bench.py) and the CPU oracle
consume exactly the bytes produced here.
"""
from .inputs import (  # noqa: F401
    x_normal,
    x_rows_normal,
    k4_uniform,
    x_int,
    k4_int,
    k4_labels,
    to_bsl,
    from_bsl,
)
from . import configs  # noqa: F401
from . import grid  # noqa: F401
