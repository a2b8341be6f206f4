"""CPU oracle for the Celerity instruction-graph coherence path (arXiv 2503.10516).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything
under `oracle/`.  The product (`paper_2503_10516_b200/`, `include/`, the
CUDA library) never imports, links or executes it, and the oracle never
imports the product.  The two share no code; the only shared module is
`workloads/` (seeded program/input descriptions, no method arithmetic).

Plain, slow, obviously-correct Python + NumPy.  Every function cites the
PAPER.md passage (P:Lnnn, section) it follows, or the DESIGN.md reading
(R0..R17) where the paper is silent.

Modules
  geometry   Box / Region (canonical form, R1-R2) / RegionMap (R3)
  program    work split (R4) and range mappers (R5)
  scheduler  task tracking + horizons (R7), lookahead (R8), IDAG
             generation: allocation (R9), coherence copies (R10),
             kernels (R11), dependencies (R12), readback / destroy (R13-14)
  cluster    virtual-node mode: N node schedulers, replicated push / await-push
             decisions, send / receive / split / await receive (R17, §3.4)
  kernels    synthetic workload arithmetic in float32 / uint32 (R16)
  simulate   byte simulator executing an instruction log over per-allocation
             arrays (R15); simulate_cluster runs every node's log with
             pilot-based receive placement
  sequential the plain definition: tasks applied in order to one global array
  invariants brute-force per-element hazard / coverage checker (R12)

Parity pins: tests/test_oracle_*.py (run with -m "not gpu").
"""
