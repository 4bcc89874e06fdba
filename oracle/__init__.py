"""ORACLE / TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference hshard executor semantics (executor.py), the
deterministic payload generator (datagen.py) and the recipe that compiles the
reference planner + a reference-primitive executor (Makefile, ref_tool.cpp ->
_ref/).  Imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, as the checker or the reported CPU
baseline.  The product (paper_2504_20490_b200) never imports it.
"""
