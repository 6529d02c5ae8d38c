"""CPU oracle of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs; never by the product package.  See lapeig_oracle.py.
"""
