"""CPU oracle for the SLICER IF codec -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg.
The product package never imports it (tests/test_no_oracle_in_product.py checks that).
"""
