"""TEST INFRASTRUCTURE ONLY: CPU parity oracle for the panel-major hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports it.
"""
