"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the CUDA path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  The product package never does.
"""
