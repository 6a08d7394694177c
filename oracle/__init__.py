"""Test infrastructure: the CPU oracle for parity checks (see iedd_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  The product (paper_2108_12574_b200) never does."""
