"""CPU oracles for the POD-2G solve path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this package.  The product (paper_2207_02543_b200) never does.
"""
