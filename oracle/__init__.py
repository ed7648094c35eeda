"""Test infrastructure: CPU oracle of the FRAM-RIR hot path (see framrir_port).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline; the product package never imports it.
"""
