"""Seeded synthetic programs and inputs shared by the oracle harness and the
GPU harness.  Holds NO arithmetic of the method (no split, mapper, region or
coherence logic, no kernel math): only descriptions of buffers, tasks and
seeded host data.  See workloads/programs.py."""
