"""CPU oracle of the reference uSR objective path -- test infrastructure only.

Imported solely by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg.  Never imported by the product package.
"""
