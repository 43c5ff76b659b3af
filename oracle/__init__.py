"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/acoustic.py header).

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs only; the product package paper_1608_03984_b200 never imports it.
"""
