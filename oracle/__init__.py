"""oracle/ — TEST INFRASTRUCTURE ONLY.

CPU restatements of the reference's evaluation of BLAS-1 expression trees
(/root/reference/pkg/src/lanevec), used as the parity checker by tests/,
by `__graft_entry__.smoke()`, by bench.py's cpu_baseline and
`--impl reference` legs (CPU timing of the reference algorithm), and by the
measurement tools tools/config_sweep.py, tools/reference_engine_timing.py
(CPU timing legs) and tools/dist_check.py (checker).

Nothing in paper_1109_1264_b200/ imports this package: the product has no
CPU evaluation path.

Modules
  restate   NumPy restatement: elementwise trees in the reference's node
            order (bit-exact), the reference engine's reduction order
            (bit-exact for a given plan), exact fsum reductions, the
            reference's scalar-loop oracles (oracle.py:26-69).
  coracle   ctypes wrapper of salt_oracle.c (C restatement, threaded).

(The chunk-keyed seeded synthetic inputs for the BASELINE configs live in
the package, paper_1109_1264_b200/synth.py: they are inputs, not a checker.)

Parity is PINNED: restate/coracle are checked in tests/test_oracle_pins.py
against golden vectors produced by the reference itself
(tests/golden/make_golden.py imports /root/reference/pkg/src in the build
container and commits the fixtures).
"""
