"""CPU ORACLE — test infrastructure only.

Imported only by tests/, __graft_entry__.smoke() and bench.py (the
cpu_baseline leg and ``--impl reference``), always as the checker or the
timed CPU baseline, never as the product path.

Two restatements of the reference FSDA path (/root/reference/pkg/src/sdakit):

* ``fsda_oracle.c`` (ctypes: ``oracle.c_oracle``) — plain C, OpenMP; row sums
  in scipy's order, every other sum in the device's canonical R256 order, so
  it agrees with the GPU bit for bit at any Krylov dimension.
* ``ref_numpy.py`` — numpy/scipy in the reference's own arithmetic (scipy
  csr/csc matvec, BLAS dots, pairwise numpy sums), for the reference-order
  checks on the GPU box, where /root/reference does not exist.

Both are pinned against the real reference's outputs by tests/golden/
(generated in the authoring container by tests/golden/make_golden.py).
"""
