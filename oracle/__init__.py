"""CPU oracle for the reference hot path -- TEST INFRASTRUCTURE ONLY.

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU legs; the
product package (paper_1703_02484_b200) never imports it.
"""
