"""TEST INFRASTRUCTURE ONLY -- the parity oracle.

Two CPU implementations of the reference hot path, both loaded with ctypes:

* ``port`` -- oracle/lib/libgdx_oracle.so, our restatement (gdx_oracle.cpp) of
  csr.cpp / graphgen.cpp / oracles.cpp and the corpus semantics.
* ``ref``  -- oracle/_ref/libgraphdsl_ref.so, the reference's own C++ sources
  compiled unchanged by oracle/Makefile, wrapped by ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package.  The product package
(paper_2401_02472_b200) never does.
"""
from .pyoracle import Port, Ref, OracleError, port_available, ref_available  # noqa: F401
