"""Write tests/golden/*.tsv from the ORACLE only (never from the CUDA path)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import schedule as S  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
os.makedirs(GOLD, exist_ok=True)
for (P, M, V) in [(2, 4, 1), (4, 8, 2)]:
    cfg = S.SchedCfg(P, M, V, llm_sched="1f1b" if V == 1 else "interleaved")
    with open(os.path.join(GOLD, f"sched_P{P}_M{M}_V{V}.tsv"), "w") as f:
        f.write(S.serialize(S.build(cfg)))
print("ok")
