"""CPU oracle of the load path — TEST INFRASTRUCTURE ONLY (see oracle.py).
Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU legs."""
