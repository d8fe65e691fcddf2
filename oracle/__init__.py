"""Test infrastructure: CPU oracles for the redsynth-b200 executor.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package — as the checker, never as the thing
measured or shipped. See numeric.h for the contract.
"""
