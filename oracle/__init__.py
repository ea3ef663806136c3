"""CPU oracle package — test infrastructure only (see flash_oracle.py header).

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs; never by the product package paper_2401_16732_b200.
"""
