"""Exhaustive searches on tiny configurations (TEST INFRASTRUCTURE).

1. min_peak_encoder_window: over ALL interleavings of EncFwd(u)/EncBwd(u)
   into the rank-0 LLM list that are dependency-safe (EncFwd(u) before F_u,
   EncBwd(u) after G_u, FIFO per kind) the minimum possible peak number of live
   encoder units.  BigMac with W = W* must attain it.
(The free-placement and cut-class searches of SURVEY §8(c) Q14 live in
tests/test_oracle_pins_r2.py with their own DES, independent of oracle/.)
"""
from __future__ import annotations

from .schedule import llm_base_schedule


def min_peak_encoder_window(P: int, M: int, V: int) -> int:
    base0 = llm_base_schedule(P, M, V)[0]
    n_u = M // P
    F = {u: base0.index(("F", u * P, 0)) for u in range(n_u)}
    G = {u: base0.index(("B", u * P + P - 1, 0)) for u in range(n_u)}
    L = len(base0)
    best = [10 ** 9]

    def rec(i, nf, nb, live, peak):
        # i: LLM ops emitted; nf/nb: EncFwd/EncBwd emitted
        if peak >= best[0]:
            return
        if i == L and nf == n_u and nb == n_u:
            best[0] = peak
            return
        # emit next LLM op if its encoder input is ready
        if i < L:
            ok = True
            for u in range(n_u):
                if F[u] == i and nf <= u:
                    ok = False
            if ok:
                rec(i + 1, nf, nb, live, peak)
        # emit EncFwd(nf)
        if nf < n_u:
            rec(i, nf + 1, nb, live + 1, max(peak, live + 1))
        # emit EncBwd(nb) if its gradient exists (G_nb emitted) and fwd done
        if nb < nf and G[nb] < i:
            rec(i, nf, nb + 1, live - 1, peak)

    rec(0, 0, 0, 0, 0)
    return best[0]
