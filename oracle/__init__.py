"""Test-infrastructure oracles for the DeFT-Flatten path (NOT the product).

* ``oracle.core``  -- ctypes wrapper over ``liboracle.so``, the plain-C
  restatement of the reference algorithms (``treeattn_oracle.c``).
* ``oracle.ref``   -- ctypes wrapper over ``_ref/libtreeattn_ref.so``, the
  unmodified reference headers compiled in place (present only where
  /root/reference existed at build time, or where the built .so travelled).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.
"""
