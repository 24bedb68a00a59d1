"""CPU oracle for BigMac's nested-pipeline training step.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import anything
under `oracle/`.  The product path (`paper_2605_25451_b200`) never imports it
and the oracle never imports the product; they share only the seeded input
generators in `synth/`.

Modules
  schedule.py  O-S: LLM base schedules, cut timeline, nesting, comm insertion,
               ring sizing, verification, statistics, serialization.
  des.py       integer discrete-event simulation of a nested schedule.
  model.py     O-N: plain fp64 forward/backward of the synthetic model,
               sequential gradient accumulation over microbatches.
  interp.py    O-N: fp64 schedule interpreter over logical ranks with runtime
               buffers (buffer-miss / leak detection).
  bruteforce.py  exhaustive placement search on tiny configs.

Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
