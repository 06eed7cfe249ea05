"""TEST INFRASTRUCTURE ONLY -- the CPU parity checker for the Jacobi-CG path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product package
(``paper_2306_17801_b200``) never imports it and has no CPU fallback.

Two libraries sit behind it (built by ``oracle/Makefile``):

* ``lib/librvk_oracle.so`` -- plain-C restatement (``rvk_oracle.c``) of the
  reference kernels (kernels_scalar.cpp:11-63), stencil assembly
   and PETSc-order Jacobi-PCG.
* ``_ref/librivulet_ref.so`` -- the reference's own kernels compiled in place
  from /root/reference/proj/src plus ``ref_shim.cpp``.  It pins the
  restatement bit-for-bit and generated ``tests/golden/``.
"""
from .oracle import *  # noqa: F401,F403
