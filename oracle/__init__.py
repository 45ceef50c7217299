"""Test infrastructure: CPU oracle for the MoE hot path (see nimg_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package. The product package never does.
"""
