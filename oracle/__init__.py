"""TEST INFRASTRUCTURE ONLY — the CPU checkers of the GPU path.

* ``oracle/_ref/libgpile_ref.so``: the unmodified reference headers behind a
  flat C shim (oracle/ref_shim.cpp), built by oracle/Makefile from
  /root/reference in this container; the built .so travels to the GPU box.
* ``oracle/_build/libgpile_oracle.so``: the plain-C restatement
  (oracle/gpile_oracle.c), pinned against the reference and the golden
  fixtures in tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package. The product path
(paper_2603_20611_b200/) never does.
"""
