"""OpenQASM 3 programs through the reference's own frontend (bounded `for` loops with
mid-circuit measurement and feedforward inside, nested if/else, register predicates),
recorded with the reference simulator's results for the B200 backend to replay.

Run in the build container (where `/root/reference` exists):

    python tests/golden/make_frontend_goldens.py

`sema.py` unrolls bounded loops statically (sema.py:640-660), so the lowered Kernel IR
the backend receives is flat; these fixtures pin that the unrolled feedforward resolves on
the device exactly as on the CPU.  Stored per program: the source, the lowered IR (mirror
JSON), the 1024-shot histogram (seed 1234) and the first 16 trajectories (keys, drawn
uniforms, final states).  Nothing is written into the reference.
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_goldens as G  # noqa: E402  (reference imports + helpers)

PROGRAMS = {
    "loop_feedforward": """OPENQASM 3.0;
include "stdgates.inc";
qubit[4] q;
bit[4] c;
bit f;
for int i in [0:3] {
  h q[i];
  c[i] = measure q[i];
  if (c[i] == 1) { x q[i]; }
}
for int i in [0:2] { cx q[i], q[i+1]; }
f = measure q[3];
""",
    "loop_nested_if": """OPENQASM 3.0;
include "stdgates.inc";
qubit[3] q;
bit[3] c;
bit[2] d;
for int r in [0:1] {
  ry(0.7) q[0]; rx(1.1) q[1]; h q[2];
  cx q[0], q[2];
  c = measure q;
  if (c >= 3) {
    if (c[0] == 1) { x q[0]; } else { h q[1]; }
  } else {
    reset q[2];
  }
  d[r] = measure q[1];
}
""",
    "loop_register_predicate": """OPENQASM 3.0;
include "stdgates.inc";
qubit[2] q;
bit[3] c;
bit e;
for int k in [0:2] {
  h q[0];
  cx q[0], q[1];
  c[k] = measure q[0];
  if (c[k] == 0) { reset q[1]; }
  rz(0.3 * (k + 1)) q[1];
  h q[1];
}
if (c != 5) { x q[1]; }
e = measure q[1];
""",
    "loop_stride_and_sdg": """OPENQASM 3.0;
include "stdgates.inc";
qubit[5] q;
bit[5] m;
for int i in [0:2:4] { h q[i]; s q[i]; }
for int i in [4:-1:1] { cx q[i-1], q[i]; }
for int i in [0:3] {
  m[i] = measure q[i];
  if (m[i] == 1) { sdg q[i + 1]; }
}
m[4] = measure q[4];
""",
}


def main():
    out = {}
    for name, src in PROGRAMS.items():
        kern = G.rsuites.compile_source(src)
        kj = G.ir.kernel_to_json(kern)
        bound = G.rkir.bind(G.to_ref(kj), [])
        hist = G.rsim.sample(bound, 1024, 1234)
        out[name] = {
            "source": src,
            "kernel": kj,
            "hist_1024_seed1234": hist.counts,
            "shots": [G.traj_record(bound, 1234, s) for s in range(16)],
        }
    G.write("frontend.json", out)


if __name__ == "__main__":
    main()
