"""fp64 CPU oracle for Nested Slice Sampling -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  It shares no code with the CUDA
product path in paper_2601_23252_b200/.
"""
