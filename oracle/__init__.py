"""ORACLE — test infrastructure only.

CPU restatement of the reference's TFT / ITFT / Algorithm-3 product
(tft_oracle.c) plus a loader for the reference's own compiled kernels
(oracle/_ref, built by ``make -C oracle ref``).  Importable only from tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs; the product package
paper_1001_5272_b200 never imports it.
"""
