"""CPU fp64 oracle for the Zero Bubble Pipeline Parallelism hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under `paper_2401_10241_b200/` may import,
call, link or execute this package.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` legs use it.

Plain, slow, obviously-correct numpy implementations written from PAPER.md
(arXiv 2401.10241), each function citing the passage it follows (P:n =
PAPER.md line n; S:n = SPEC.md line n; SURVEY §x = the reading chosen in
SURVEY.md and listed in DESIGN.md).  The oracle shares no code with the CUDA
path; the only shared module is `zb_synth` (seeded inputs, no arithmetic).

Modules
  model     GPT-style stage math: F, unsplit backward, split B / W.
  schedule  1F1B / ZB-H1 / ZB-H2 builders, AUTO heuristic + grid search,
            simulator, memory / slot accounting, closed forms (P:57-142,
            P:286).
  optim     AdamW step and in-place rollback (Algorithm 1),
            post-validation protocol and synchronous baseline.

Pins (tests/test_oracle_*.py): torch fp64 autograd and finite differences
for the model; Table 2 closed forms, Table 4 printed bubble rates, per-stage
memory expressions and brute-force optima for the schedules; Algorithm 1
hand example and round-trip for the optimizer; fault corpus vs synchronous
baseline for post-validation.  Parity unpinned: the exact AUTO pass ORDER
(only its simulated cost is pinned by Table 4).
"""
