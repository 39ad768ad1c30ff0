"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a, loads without a
GPU, exports every symbol include/asyncep.h declares, and its pure host functions
(sizes, config validation, Eq. 1) agree with the oracle.  No device compute here."""
import ctypes
import os
import re
import subprocess

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def A():
    from paper_2605_02960_b200 import build
    build.build()
    from paper_2605_02960_b200 import asyncep
    return asyncep


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "asyncep.h")).read()
    return sorted(set(re.findall(r"ASYNCEP_API\s+[\w\s\*]+?\b(asyncep_\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_symbols()
    for required in ("asyncep_init", "asyncep_prefetch_layer", "asyncep_moe_forward", "asyncep_saturation_T"):
        assert required in names


def test_library_exports_every_declared_symbol(A):
    lib = ctypes.CDLL(A.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (asyncep_\w+)", out))
    assert set(declared_symbols()) <= exported
    assert A.asyncep_abi_version() == 1


def test_library_is_sm100a_code(A):
    out = subprocess.run(["cuobjdump", "--list-elf", A.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", A.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass, "no tcgen05 MMA in the binary"
    assert "UTMALDG" in sass, "no TMA loads in the binary"
    assert "LDTM" in sass, "no TMEM loads in the binary"


def test_hot_kernels_do_not_spill(A):
    """The production-path kernels keep their state in registers (cuobjdump -res-usage STACK:0): a
    local-memory spill in a tensor-core pipeline role (e.g. a runtime-indexed register array in an
    epilogue) costs the GEMM its issue slots silently.  (Debug / fallback kernels -- the SIMT
    router and GEMM, the destination-list FP8 quantisation -- may use local arrays.)"""
    out = subprocess.run(["cuobjdump", "-res-usage", A.LIB_PATH], capture_output=True, text=True).stdout
    funcs = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", out)
    assert funcs, out[:500]
    hot = ("gemm_tc_kernel", "combine_kernel", "perm_hist", "perm_scan", "perm_scatter", "quant_tokens",
           "act_quant", "gather_copy", "flash_attn4", "rmsnorm", "qk_rope", "v_transpose")
    assert any(h in f for f, _, _ in funcs for h in hot)
    spills = [(f, st) for f, reg, st in funcs if int(st) != 0 and any(h in f for h in hot)]
    assert not spills, spills


def test_sizes_and_config_validation(A):
    cfg = A.make_config(8, 128, 8, 4096, 1536, world_size=8, max_tokens=32768)
    assert A.asyncep_expert_bytes(cfg) == 3 * 4096 * 1536 * 2
    assert A.asyncep_slot_bytes(cfg) == 4_831_838_208  # SURVEY.md appendix (BF16 layer)
    assert A.asyncep_shard_bytes(cfg) == 4_831_838_208 // 8
    assert A.asyncep_workspace_size(cfg) > 32768 * 8 * (4096 + 1536) * 2
    bad = [dict(num_experts=100, world_size=8),  # E % N != 0
           dict(hidden=4000), dict(ffn=1000), dict(top_k=0), dict(top_k=17), dict(gamma=0.5),
           dict(max_tokens=0)]
    for b in bad:
        kw = dict(num_layers=8, num_experts=128, top_k=8, hidden=4096, ffn=1536, world_size=8, max_tokens=1024)
        kw.update(b)
        c = A.make_config(kw.pop("num_layers"), kw.pop("num_experts"), kw.pop("top_k"), kw.pop("hidden"),
                          kw.pop("ffn"), **kw)
        with pytest.raises(A.AsyncEPError):
            A.asyncep_workspace_size(c)


@pytest.mark.parametrize("N", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype,b,F", [(0, 2, 1.42e15), (1, 1, 2.84e15)])
def test_saturation_T_matches_oracle(A, N, dtype, b, F):
    cfg = A.make_config(8, 128, 8, 4096, 1536, expert_dtype=dtype, world_size=N, max_tokens=1, gamma=1.2)
    t, f = A.asyncep_saturation_T(cfg, F, 7.5e11)
    t0, f0 = oracle.saturation_T(128, 8, 4096, 1536, b, N, float(ctypes.c_float(1.2).value), F, 7.5e11)
    assert t == pytest.approx(t0, rel=1e-12) and f == pytest.approx(f0, rel=1e-12)
    if N == 1:
        assert t == 0.0


def test_calibrated_T_matches_oracle(A):
    """App. B.4 Eq. 3 through the C ABI vs the oracle (and SPEC's worked example)."""
    for g, te, tc, c in ((1.2, 2.0, 1.0, 1e12), (1.2, 0.5, 1.0, 7.0), (1.5, 3.3, 1.1, 4e13), (1.0, 1.0, 1.0, 5.0)):
        assert A.asyncep_calibrated_T(g, te, tc, c) == pytest.approx(oracle.calibrated_T(g, te, tc, c), rel=1e-15)
    assert A.asyncep_calibrated_T(1.2, 2.0, 1.0, 1e12) == pytest.approx(2.4e12, rel=1e-15)
    with pytest.raises(A.AsyncEPError):
        A.asyncep_calibrated_T(0.9, 1.0, 1.0, 1.0)


def test_ep_plan_layout(A):
    """DP x EP exchange plan: rank d's experts are one contiguous padded
    range of the sender's X_perm; the receive buffer is source-major, expert-ordered."""
    import numpy as np
    cfg = A.make_config(1, 8, 2, 256, 256, world_size=4, rank=1, max_tokens=1024)
    sc = np.array([5, 0, 300, 256, 1, 2, 0, 513], np.int32)
    rc = np.array([1, 2, 3, 4, 0, 0, 257, 255], np.int32)
    p = A.asyncep_ep_plan(cfg, sc, rc)
    pad = lambda n: (n + 255) // 256 * 256
    assert list(p["send_rows"]) == [pad(5) + pad(0), pad(300) + pad(256), pad(1) + pad(2), pad(0) + pad(513)]
    assert list(p["send_off"]) == list(np.concatenate([[0], np.cumsum(p["send_rows"])[:-1]]))
    assert list(p["recv_rows"]) == [pad(1) + pad(2), pad(3) + pad(4), 0, pad(257) + pad(255)]
    assert p["group_off"][-1] == p["recv_total"] == sum(p["recv_rows"])
    assert all(o % 256 == 0 for o in p["group_off"])
