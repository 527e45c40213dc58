"""TEST INFRASTRUCTURE ONLY: the CPU oracle (see oracle/README.md).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arms may import this package, and only as the checker or the timed CPU
baseline — never as the product path.
"""
