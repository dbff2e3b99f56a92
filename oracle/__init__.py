"""ORACLE — test infrastructure only (CPU restatement of the reference hot path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this package; the product (paper_2405_02187_b200) never does.
"""
