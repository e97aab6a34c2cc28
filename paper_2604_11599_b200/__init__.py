"""B200-native state-vector backend for the qasm2cudaq simulator target.

Drop-in for `qasm2cudaq.sim` (reference: /root/reference/pkg/src/qasm2cudaq/sim.py).
See DESIGN.md.
"""

__version__ = "0.1.0"
