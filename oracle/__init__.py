"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke, bench.py cpu_baseline)."""
