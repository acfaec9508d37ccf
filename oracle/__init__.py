"""CPU oracle for the iHDG-II sweep -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs.  Never imported by the product package.
"""
