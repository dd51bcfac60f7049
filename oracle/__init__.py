"""Test-infrastructure package: CPU oracle for the state-vector hot path.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this; the product (paper_2509_04955_b200) never does.  See oracle/oracle.h.
"""
