"""Parity oracles — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
arm may import this package, and only as the checker. The product
(paper_2508_12627_b200) never imports it.
"""
