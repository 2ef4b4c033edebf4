"""CPU oracle for the APEX retrieval path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference legs, as the checker or the timed CPU baseline; never by
the product package.  See scan_oracle.py for the restated reference functions
(with file:line citations) and tests/golden/ for the fixtures that pin it.
"""
