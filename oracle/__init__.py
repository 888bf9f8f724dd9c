"""CPU oracle for the Picker hot path -- TEST INFRASTRUCTURE, not product code.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import anything under oracle/.  The product package
paper_2410_23661_b200 never imports it, and it never imports the product
package; both read the same seeded inputs from tracegen/ (which holds no
validation arithmetic).

Parity pins: see tests/test_oracle_pins.py (paper examples in tests/golden/,
brute-force kernel simulations, closed forms, invariants).  Parity unpinned:
none of the functions here; the paper's aggregate accuracy numbers (18.54 % FN,
Table 3) are not reproducible without its kernels and are not claimed.
"""
from .picker_oracle import *  # noqa: F401,F403
