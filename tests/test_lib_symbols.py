"""The C-ABI library loads on a CPU-only host and exports every function that
include/*.h declares (no compute calls).  Also checks the parameter layout
the library computes against synth.param_specs (host logic only)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for h in ("bigmac.h", "bigmac_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:bm_status|void|int64_t|const char\*)\s+(bm_\w+)\s*\(", src, flags=re.M):
            names.append(m.group(1))
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_2605_25451_b200 import _lib as L
    lib = L.lib()
    names = declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(L.SIGNATURES), set(names) ^ set(L.SIGNATURES)
    assert L.MISSING == []


def test_library_is_sm100a():
    import subprocess
    so = os.path.join(ROOT, "paper_2605_25451_b200", "libbigmac.so")
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", so], capture_output=True, text=True)
    assert "sm_100a" in r.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA loads
    assert "LDTM" in sass             # tcgen05.ld (TMEM -> registers)


def expected_layers(L, P, V, last, s, explicit=None):
    """bigmac.h "LLM layer partition": layers of virtual stage s."""
    PV = P * V
    if explicit:
        start = sum(explicit[:s])
        return list(range(start, start + explicit[s]))
    if last == 0 or PV == 1:
        n = L // PV
        return list(range(s * n, (s + 1) * n))
    if s == PV - 1:
        return list(range(L - last, L))
    counts = [(L - last) // (PV - 1) + (1 if i < (L - last) % (PV - 1) else 0) for i in range(PV - 1)]
    start = sum(counts[:s])
    return list(range(start, start + counts[s]))


@pytest.mark.parametrize("head,last", [("auto", 0), ("last_stage", 0), ("dp_shard", 0), ("auto", 1), ("auto", 2)])
@pytest.mark.parametrize("P,V,rank", [(1, 1, 0), (2, 1, 0), (2, 1, 1), (4, 1, 3), (2, 2, 0), (2, 2, 1), (1, 4, 0)])
def test_param_layout_matches_model(P, V, rank, head, last):
    from synth import get_config, param_specs
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200 import schedule as BS
    from paper_2605_25451_b200.runtime import model_cfg
    cfg = get_config("C1", P=P, M=2 * P, V=V)
    if last and cfg.L - last < P * V - 1:
        pytest.skip("partition needs a layer per virtual stage")
    explicit = None
    if last == 2 and P * V == 2:     # also an explicit partition (stage_layers)
        explicit = [1, 3]
    mc = model_cfg(cfg, "bf16", head_place=head, last_stage_layers=last, stage_layers=explicit)
    sc = BS.make_cfg(P, 2 * P, V)
    head_dp = head == "dp_shard"   # bigmac.h bm_head_place (auto = last stage)
    n, tot, dp = C.c_int32(), C.c_int64(), C.c_int64()
    L.call("bm_param_count", C.byref(mc), C.byref(sc), rank, C.byref(n), C.byref(tot), C.byref(dp))
    specs = {nm: shp for nm, shp, _ in param_specs(cfg)}
    got = {}
    prev_end = 0
    for i in range(n.value):
        pi = L.ParamInfo()
        L.call("bm_param_info_get", C.byref(mc), C.byref(sc), rank, i, C.byref(pi))
        nm = pi.name.decode()
        shp = specs[nm]
        rows, cols = shp[0], (shp[1] if len(shp) > 1 else 1)
        assert (pi.rows, pi.cols) == (rows, cols)
        assert pi.offset >= prev_end and pi.offset % 64 == 0 and pi.ld >= cols and pi.ld % (1 if cols == 1 else 8) == 0
        prev_end = pi.offset + rows * pi.ld
        got[nm] = pi.kind
    my_layers = {l for c in range(V) for l in expected_layers(cfg.L, P, V, last, c * P + rank, explicit)}
    for nm in specs:
        if nm.startswith(("enc.", "gen.")):
            assert got.get(nm) == 0, nm            # DP params on every rank
        elif nm == "llm.embed":
            assert (nm in got) == (rank == 0)
        elif nm == "llm.head" and head_dp:
            assert got.get(nm) == 0, nm            # DP-sharded head: a DP param on every rank
        elif nm in ("llm.final_norm", "llm.head"):
            assert (nm in got) == (rank == P - 1)
        else:
            l = int(nm.split(".")[1][5:])
            assert (nm in got) == (l in my_layers), nm
    assert prev_end <= tot.value and dp.value <= tot.value


def test_layer_partition_examples_and_errors():
    # (5, 4, 4, 3) at L = 16, P = 4 and (3, 2, 2, 2, 2, 2, 2, 1) at P = 8
    assert [len(expected_layers(16, 4, 1, 3, s)) for s in range(4)] == [5, 4, 4, 3]
    assert [len(expected_layers(16, 8, 1, 1, s)) for s in range(8)] == [3, 2, 2, 2, 2, 2, 2, 1]
    from synth import get_config
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200 import schedule as BS
    from paper_2605_25451_b200.runtime import model_cfg
    cfg = get_config("C1", P=2, M=4, V=1)
    n, tot, dp = C.c_int32(), C.c_int64(), C.c_int64()
    for bad in (cfg.L, -1):
        mc = model_cfg(cfg, "bf16", last_stage_layers=bad)
        with pytest.raises(L.BigMacError):
            L.call("bm_param_count", C.byref(mc), C.byref(BS.make_cfg(2, 4, 1)), 0, C.byref(n), C.byref(tot), C.byref(dp))
    mc = model_cfg(cfg.replace(L=5), "bf16")       # L % (P V) != 0 needs an explicit partition
    with pytest.raises(L.BigMacError):
        L.call("bm_param_count", C.byref(mc), C.byref(BS.make_cfg(2, 4, 1)), 0, C.byref(n), C.byref(tot), C.byref(dp))
    mc = model_cfg(cfg.replace(L=5), "bf16", last_stage_layers=2)
    L.call("bm_param_count", C.byref(mc), C.byref(BS.make_cfg(2, 4, 1)), 0, C.byref(n), C.byref(tot), C.byref(dp))
    for bad in ([1, 2], [4, 0], [2, 2, 1]):      # sum != L, empty stage, beyond P*V ([0, ...] = unset)
        mc = model_cfg(cfg, "bf16", stage_layers=bad)
        with pytest.raises(L.BigMacError):
            L.call("bm_param_count", C.byref(mc), C.byref(BS.make_cfg(2, 4, 1)), 0, C.byref(n), C.byref(tot), C.byref(dp))
    mc = model_cfg(cfg, "bf16", head_place="dp_shard")
    with pytest.raises(L.BigMacError):       # the DP-sharded head rides on DP-sharded generator ops
        L.call("bm_param_count", C.byref(mc), C.byref(BS.make_cfg(2, 4, 1, gen_place="last_stage")), 0,
               C.byref(n), C.byref(tot), C.byref(dp))


@pytest.mark.parametrize("P", [1, 2, 4])
def test_fsdp_shards_partition_the_dp_parameters(P):
    """FSDP (bm_model_cfg.fsdp), host logic only: the ranks' shards
    [lo_r, hi_r) tile the DP parameter prefix exactly once, each rank's weights buffer
    shrinks by the unowned DP elements, and the unsupported combinations are rejected."""
    from synth import get_config
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200 import schedule as BS
    from paper_2605_25451_b200.runtime import model_cfg
    cfg = get_config("C1", P=P, M=2 * P, V=1)
    sched = BS.build(P, 2 * P, 1)
    shards, sizes = [], []
    for r in range(P):
        out = []
        for mode in ("off", "pull"):
            mc = model_cfg(cfg, "bf16", fsdp=mode)
            h = C.c_void_p()
            L.call("bm_ctx_create", C.byref(mc), sched.handle, r, C.byref(h))
            sz = L.CtxSizes()
            L.call("bm_ctx_sizes_get", h, C.byref(sz))
            lo, hi = C.c_int64(), C.c_int64()
            L.call("bm_ctx_dp_shard", h, C.byref(lo), C.byref(hi))
            out.append((sz.weight_bytes, lo.value, hi.value))
            L.lib().bm_ctx_destroy(h)
        (w_off, lo0, hi0), (w_fsdp, lo, hi) = out
        dp = hi0 - lo0
        assert lo0 == 0 and dp > 0
        assert w_off - w_fsdp == (dp - (hi - lo)) * 2
        shards.append((lo, hi))
    assert shards[0][0] == 0 and shards[-1][1] == dp
    assert all(shards[i][1] == shards[i + 1][0] for i in range(P - 1))
    assert all(lo % 4 == 0 for lo, _ in shards)
    mc = model_cfg(cfg, "bf16", fsdp="pull", head_place="dp_shard")
    h = C.c_void_p()
    assert L.lib().bm_ctx_create(C.byref(mc), sched.handle, 0, C.byref(h)) == 1   # BM_E_INVALID


@pytest.mark.parametrize("P,V,units", [(2, 1, [3, 5]), (2, 1, [5, 3]), (4, 1, [3, 2, 2, 1]), (2, 2, [1, 3, 2, 2]),
                                       (4, 1, [1, 1, 1, 5])])
def test_param_layout_half_layer_units(P, V, units):
    """stage_halves (bigmac.h, reading R24): unit 2l = layer l's norm + gate_up, unit
    2l + 1 = its down; every rank holds exactly the parameters of its units, each
    LLM parameter lives on one rank."""
    from synth import get_config
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200 import schedule as BS
    from paper_2605_25451_b200.runtime import model_cfg
    cfg = get_config("C1", P=P, M=2 * P, V=V)
    assert sum(units) == 2 * cfg.L
    mc = model_cfg(cfg, "bf16", stage_layers=units, stage_halves=True)
    sc = BS.make_cfg(P, 2 * P, V)
    owner = {}
    for rank in range(P):
        n, tot, dp = C.c_int32(), C.c_int64(), C.c_int64()
        L.call("bm_param_count", C.byref(mc), C.byref(sc), rank, C.byref(n), C.byref(tot), C.byref(dp))
        for i in range(n.value):
            pi = L.ParamInfo()
            L.call("bm_param_info_get", C.byref(mc), C.byref(sc), rank, i, C.byref(pi))
            nm = pi.name.decode()
            if nm.startswith("llm.layer"):
                assert nm not in owner, nm
                owner[nm] = rank
    for s in range(P * V):
        rank = s % P
        for u in range(sum(units[:s]), sum(units[:s + 1])):
            l, half = divmod(u, 2)
            names = [f"llm.layer{l}.down"] if half else [f"llm.layer{l}.norm", f"llm.layer{l}.gate_up"]
            for nm in names:
                assert owner.pop(nm) == rank, (nm, s)
    assert not owner


def test_half_layer_units_errors():
    from synth import get_config
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200 import schedule as BS
    from paper_2605_25451_b200.runtime import model_cfg
    cfg = get_config("C1", P=2, M=4, V=1)
    n, tot, dp = C.c_int32(), C.c_int64(), C.c_int64()
    for bad in ([4, 3], [8, 0], None):       # sum != 2L, empty stage, no explicit partition
        mc = model_cfg(cfg, "bf16", stage_layers=bad, stage_halves=True)
        with pytest.raises(L.BigMacError):
            L.call("bm_param_count", C.byref(mc), C.byref(BS.make_cfg(2, 4, 1)), 0, C.byref(n), C.byref(tot), C.byref(dp))


def test_executor_rejects_cp_schedules():
    """bm_ctx_create runs llm_cp = enc_cp = 1 only (the CP schedule is host-level, R25)."""
    from synth import get_config
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200 import schedule as BS
    from paper_2605_25451_b200.runtime import model_cfg
    cfg = get_config("C1", P=2, M=8, V=1)
    mc = model_cfg(cfg, "bf16")
    sched = BS.build(2, 8, 1, llm_cp=2, gen_place="last_stage")
    h = C.c_void_p()
    with pytest.raises(L.BigMacError) as e:
        L.call("bm_ctx_create", C.byref(mc), sched.handle, 0, C.byref(h))
    assert e.value.code == 1 and "CP" in str(e.value)
