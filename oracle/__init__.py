"""NanoSpec CPU oracle -- TEST INFRASTRUCTURE (see oracle/oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg /
``--impl reference`` may import this package.
"""
