"""CPU oracle package -- TEST INFRASTRUCTURE ONLY.

Import allowed from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  The product package ``paper_2604_03950_b200`` never
imports this.
"""
