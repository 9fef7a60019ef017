"""oracle — CPU checkers for the MLMC sample path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this package. The product (paper_2306_13493_b200/) must never import it.
"""
