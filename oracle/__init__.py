"""TEST INFRASTRUCTURE ONLY: the fp64 CPU oracle (see oracle/oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.
"""
