"""Seeded synthetic workload generators (C1-C5) shared by tests, bench and oracle callers.
Holds no arithmetic of the method itself."""
