"""CPU-only checks of the product boundary: the C-ABI library loads and
exports every symbol include/tsq.h declares, host-side API semantics
(config validation, RNG, error mapping) -- no compute calls without a GPU."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1505_00558_b200 as T
from paper_1505_00558_b200 import _native as N
from paper_1505_00558_b200.build import LIB, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    text = open(os.path.join(ROOT, "include", "tsq.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tsq_[a-z_]+)\s*\(", text)))


def test_library_builds_and_exports_header_symbols():
    build()
    assert os.path.exists(LIB)
    lib = ctypes.CDLL(LIB)
    declared = _header_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(N.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_abi():
    lib = N.lib()
    assert lib.tsq_abi_version() == 2
    assert N.status_str(N.TSQ_ERR_BUSY) == "sorter instance is not reentrant"
    assert N.status_str(N.TSQ_OK) == "ok"


def test_workspace_bytes_scales():
    lib = N.lib()
    a = lib.tsq_workspace_bytes(1 << 20, N.TSQ_I32, N.TSQ_NONE)
    b = lib.tsq_workspace_bytes(1 << 24, N.TSQ_I32, N.TSQ_NONE)
    c = lib.tsq_workspace_bytes(1 << 20, N.TSQ_U64, N.TSQ_U32)
    assert 4 << 20 <= a < 6 << 20       # one n*4 partner + small queues
    assert 64 << 20 <= b < 80 << 20
    assert c >= (1 << 20) * 16          # keys partner + payload partner + side buffer
    assert lib.tsq_workspace_bytes(1 << 20, 99, 0) == 0


def test_abi_struct_sizes_match_header():
    # tsq_params: 8 + 7*4 (+4 pad) + 2 pointers + 1*8 ; tsq_stats: 20 u64 + 2 floats;
    # tsq_stage_record: 5*8 + 2*4 (static_asserts in tsq_capi.cu pin the C side)
    assert ctypes.sizeof(N.TsqParams) == 64
    assert ctypes.sizeof(N.TsqStats) == 20 * 8 + 8
    assert ctypes.sizeof(N.TsqStageRecord) == 48
    src = open(os.path.join(ROOT, "paper_1505_00558_b200", "csrc", "tsq_capi.cu")).read()
    assert "sizeof(tsq_params) == 64" in src and "sizeof(tsq_stats) == 168" in src


def test_sortconfig_validation_matches_reference():
    # reference config.py:28-42
    with pytest.raises(ValueError):
        T.SortConfig(insertion_threshold=2)
    with pytest.raises(ValueError):
        T.SortConfig(medof3_max_n=700)
    with pytest.raises(ValueError):
        T.SortConfig(reverse_tolerance=-1)
    with pytest.raises(ValueError):
        T.SortConfig(late_swap_byte_threshold=0)
    T.SortConfig(insertion_threshold=3)
    with pytest.raises(ValueError):
        T.GpuConfig(small_threshold=40953)
    with pytest.raises(ValueError):
        T.GpuConfig(small_threshold=-1)
    assert T.GpuConfig().small_threshold == 0  # auto: the measured per-type default
    with pytest.raises(ValueError):
        T.GpuConfig(max_depth=1)
    assert T.GpuConfig().max_depth == 0  # auto: max(24, 2 log2 n)
    T.GpuConfig(max_depth=2)


def test_rng_matches_reference_kats():
    r = T.MitigationRng(1)
    T.rng_next(r)
    assert r.zgen == 16807
    T.rng_next(r)
    assert r.zgen == 282475249
    for _ in range(100):
        T.rng_next(r)
        assert 0.5 <= r.dran < 1.5 and r.dran2 == 1 + r.dran
    assert T.MitigationRng(0).zgen != 0


def test_rng_matches_golden():
    from conftest import load_golden
    for case in load_golden("rng.json"):
        r = T.MitigationRng(case["seed"])
        for zgen, dran, dran2 in case["seq"]:
            r.next()
            assert (r.zgen, r.dran, r.dran2) == (zgen, dran, dran2)


def test_registry_signature():
    fn = T.get_algorithm("tristate")
    assert fn is T.REGISTRY["tristate"]
    with pytest.raises(KeyError):
        T.get_algorithm("nope")


def test_trivial_inputs_need_no_device():
    # n <= 1 returns before touching CUDA (core.py:1592-1593 semantics)
    for ar in ([], [7]):
        got = list(ar)
        st = T.Sorter().sort_with_stats(got)
        assert got == ar and st.comparisons == 0 and st.element_writes == 0


def test_rejects_custom_comparator_without_fallback():
    with pytest.raises(TypeError):
        T.Sorter().sort([3, 1, 2], cmp=lambda a, b: (a > b) - (a < b))
    with pytest.raises(TypeError):  # the late-swap path has no comparator fallback either
        T.Sorter().sort([3, 1, 2], cmp=lambda a, b: (a > b) - (a < b), element_size=400)
    with pytest.raises(TypeError):
        T.Sorter().sort(["a", "b", "c"])


# ---- late swapping (bigelem.py): host-side permutation semantics -----------

def test_apply_identity_zero_moves():
    ar = list(range(5))
    assert T.apply_permutation(ar, T.Permutation((0, 1, 2, 3, 4))) == 0
    assert ar == [0, 1, 2, 3, 4]


def test_apply_single_two_cycle():
    ar = [1, 0, 2]
    assert T.apply_permutation(ar, T.Permutation((1, 0, 2))) == 3
    assert ar == [0, 1, 2]


def test_apply_full_reversal_n6():
    ar = [5, 4, 3, 2, 1, 0]
    assert T.apply_permutation(ar, T.Permutation((5, 4, 3, 2, 1, 0))) == 9
    assert ar == [0, 1, 2, 3, 4, 5]


def test_permutation_length_mismatch():
    with pytest.raises(ValueError):
        T.apply_permutation([1, 2], T.Permutation((0, 1, 2)))


def test_cycle_move_count_matches_reference_walk():
    """moves = sum(c + 1) over nontrivial cycles (bigelem.py:48-76), from
    the pointer-jumping cycle count, on random permutations."""
    from paper_1505_00558_b200.bigelem import cycle_moves
    rng = np.random.default_rng(3)
    for n in (0, 1, 2, 7, 64, 1000, 4097):
        p = rng.permutation(n)
        if n > 10:
            p[: n // 3] = np.arange(n // 3)  # fixed points
            p[n // 3:] = rng.permutation(np.arange(n // 3, n))
        seen = np.zeros(n, bool)
        want = cyc = 0
        for i in range(n):
            if seen[i]:
                continue
            c, j = 0, i
            while not seen[j]:
                seen[j] = True
                j = p[j]
                c += 1
            if c > 1:
                want += c + 1
                cyc += 1
        assert cycle_moves(p) == (want, cyc)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        T.Sorter().sort([3, 1, 2])


def test_reentrancy_flag():
    s = T.Sorter()
    s._active = True
    with pytest.raises(RuntimeError, match="not reentrant"):
        s.sort([2, 1])
    with pytest.raises(RuntimeError):
        s.free_temp_storage()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1505_00558_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.replace("oracle/", "").lower() or f == "core.py" \
                    and "import oracle" not in text, f
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "tsq_oracle" not in text, f


def test_workloads_generators_small():
    import workloads as W
    for fam in W.FAMILIES:
        k, p = W.generate(fam, 4096)
        assert k.size == 4096
        assert (p is None) == (not W.FAMILIES[fam][1])
    k, _ = W.generate("normal_f64", 100000)
    assert not np.isnan(k).any() and not (np.signbit(k) & (k == 0)).any()


def test_battery_generators_match_reference():
    """tests/battery.py (the reference's datagen restated) reproduces the
    reference's own battery inputs (tests/golden/battery.json, written by
    tests/golden/make_battery.py from tsqsort.datagen)."""
    import hashlib
    from battery import battery_cells, generate
    from conftest import load_golden
    g = load_golden("battery.json")
    sha = lambda a: hashlib.sha256(np.asarray(a, dtype=np.int64).tobytes()).hexdigest()[:16]
    sm = g["small"]
    for d, r in battery_cells():
        a = generate(d, r, sm["n"], sm["arange"], sm["seed"])
        assert sha(a) == sm["cells"][f"{d}/{r}"], (d, r)
    for key in ("random/fort", "shuffle/dither", "organpipes/reversed", "stagger/sorted"):
        d, r = key.split("/")
        a = generate(d, r, g["n"], g["arange"], g["seed"])
        assert sha(a) == g["cells"][key]["input_sha"], key
        assert sha(np.sort(a)) == g["cells"][key]["sorted_sha"], key
