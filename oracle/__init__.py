"""Parity checker for the CUDA path. TEST INFRASTRUCTURE ONLY.

- coconet_oracle : numpy/C restatement of the reference's arithmetic
- ref            : the unmodified reference (ccopt) compiled in place
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this package; the product package never does.
"""
