"""CPU-side checks of the C ABI: libnmspmm.so builds for sm_100a, loads, exports
every symbol include/*.h declares, and rejects bad arguments synchronously.
No kernel is launched here (there is no GPU in the dev container); without a
device the compute entry points must fail loudly with NM_ERR_CUDA (no CPU
fallback)."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w]*\s*\**\s*(nm_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def L():
    from paper_2503_01253_b200 import build, nmspmm
    build.build()
    return nmspmm.lib()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["nm_compress", "nm_spmm", "nm_decompress", "nm_validate", "nm_plan_query", "nm_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(L):
    from paper_2503_01253_b200 import nmspmm
    out = subprocess.run(["nm", "-D", "--defined-only", nmspmm.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT\s+(nm_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    assert set(nmspmm.EXPORTS) <= set(declared_functions())


def test_library_is_sm100a_only(L):
    from paper_2503_01253_b200 import nmspmm
    out = subprocess.run(["cuobjdump", "--list-elf", nmspmm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if line.strip())


def test_sass_uses_tma(L):
    from paper_2503_01253_b200 import nmspmm
    sass = subprocess.run(["cuobjdump", "-sass", nmspmm.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # TMA loads in the tiled kernels


def test_version_and_config(L):
    assert L.nm_version().decode().startswith("nmspmm")
    assert L.nm_check_config(2, 4, 4) == 0
    for N, M, Lv in [(0, 4, 1), (5, 4, 1), (1, 257, 1), (1, 4, 0)]:
        assert L.nm_check_config(N, M, Lv) == 1
    assert b"N:M" in L.nm_last_error()


def test_argument_errors_are_synchronous(L):
    P = ctypes.c_void_p(16)  # never dereferenced: the shape check fails first
    # k % M != 0
    assert L.nm_spmm(P, P, P, P, 8, 8, 6, 2, 4, 1, 0, 0, 0, None) == 2
    # n % L != 0
    assert L.nm_spmm(P, P, P, P, 8, 6, 8, 2, 4, 4, 0, 0, 0, None) == 2
    # bad config
    assert L.nm_spmm(P, P, P, P, 8, 8, 8, 5, 4, 1, 0, 0, 0, None) == 1
    # fp32 operands with bf16 C is unsupported -- but only reported once a device exists;
    # NULL pointers
    assert L.nm_spmm(None, None, None, None, 8, 8, 8, 2, 4, 1, 0, 0, 0, None) == 8
    # empty problem is a no-op
    assert L.nm_spmm(None, None, None, None, 0, 8, 8, 2, 4, 1, 0, 0, 0, None) == 0
    assert L.nm_compress(P, 0, 6, 8, 2, 4, 1, P, 0, P, None) == 2


def test_no_cpu_fallback_without_device(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    P = ctypes.c_void_p(256)
    st = L.nm_spmm(P, P, P, P, 8, 8, 8, 2, 4, 1, 0, 0, 0, None)
    assert st == 7 and b"no CUDA device" in L.nm_last_error()


def test_plan_query_model(L):
    from paper_2503_01253_b200 import nmspmm
    import torch
    p = nmspmm.nm_plan_query(4096, 4096, 4096, 16, 32, 32, torch.float32)
    assert p["kernel"] == 1 and p["bm"] == 128 and p["bk"] == 64 and p["bkw"] == 32
    assert p["flops"] == 2 * 4096 * 4096 * 2048
    assert p["bytes"] == 4 * 4096 * 4096 + 4 * 2048 * 4096 + 2048 * 128 + 4 * 4096 * 4096
    assert p["bound"] == 0  # FMA-bound
    q = nmspmm.nm_plan_query(256, 255, 256, 2, 4, 3, torch.float32)
    assert q["kernel"] == 0  # L % 4 != 0 -> generic


# The SIMT kernel's split choice (nm_plan_query.split, simt_split_factor) pinned to the fastest
# split factor measured on B200 for each shape (profiles/r02c_simt_streamk.txt, table 1: kernel
# time under NM_SIMT_SPLIT = 1..4; 148 SMs, 296 resident CTAs).
SPLIT_MEASURED = [
    # (m, n, k, N, M, L), fastest S, why
    ((2048, 5120, 5120, 4, 32, 32), 3),    # 640 tiles: a 48-tile tail -> 144 lone CTAs
    ((256, 22016, 8192, 4, 32, 32), 3),    # 344 tiles: 48-tile tail
    ((2048, 2752, 8192, 4, 32, 32), 2),    # cfg4-65B 8-GPU shard, 352 tiles: 56-tile tail
    ((2048, 13824, 5120, 4, 32, 32), 1),   # 1728 tiles: 248-tile tail is most of a wave
    ((4096, 4096, 4096, 16, 32, 32), 1),   # cfg2: 1024 tiles, 136-tile tail
    ((256, 13824, 5120, 4, 32, 32), 1),    # 216 tiles, sub-wave: a split would double up SMs
    ((4096, 512, 4096, 16, 32, 32), 1),    # cfg2 8-GPU shard: 128 tiles, one per SM already
    ((2048, 1376, 4096, 8, 32, 32), 2),    # cfg3-75% 8-GPU shard: 176 tiles -> 296 + 56 lone
    ((1024, 1024, 1024, 16, 32, 32), 2),   # 64 tiles x 2 = 128 lone CTAs, 256 rows each
    ((1024, 1024, 1024, 4, 32, 32), 1),    # 64 tiles, 128 rows: too short to split
    ((2048, 2048, 2048, 16, 32, 32), 1),   # 256 tiles, sub-wave
]


@pytest.mark.parametrize("cfg,best", SPLIT_MEASURED)
def test_plan_simt_split_matches_measured_best(L, monkeypatch, cfg, best):
    """The split rule of the 128-row tile (the measurements above were taken with it)."""
    from paper_2503_01253_b200 import nmspmm
    import torch
    monkeypatch.setenv("NM_SIMT_BM", "128")
    p = nmspmm.nm_plan_query(*cfg, torch.float32)
    assert p["kernel"] == 1
    assert p["split"] == best, p
    m, n = cfg[:2]
    tiles = -(-m // 128) * -(-n // 128)
    assert p["grid"] == tiles - p["split_tiles"] + p["split_tiles"] * p["split"]
    assert abs(p["waves"] - p["grid"] / 296) < 1e-9


# The 64-row tile's split (small grids whose split CTAs all run alone) pinned to the fastest
# measured S (profiles/r02v_simt_small_split.txt, NM_SIMT_BM=64 with NM_SIMT_SPLIT 1..4).
SPLIT64_MEASURED = [
    ((512, 1024, 1024, 16, 32, 32), 2),    # 64 tiles: 31.1 vs 39.0 us
    ((512, 512, 512, 16, 32, 32), 2),      # 32 tiles, w = 256: 25.2 vs 27.5
    ((1024, 1024, 1024, 16, 32, 32), 1),   # 128 tiles: 2 x 128 > 148 SMs (46.0 vs 39.6)
    ((1024, 1024, 1024, 4, 32, 32), 1),    # 23.4 vs 30.4
    ((256, 256, 256, 2, 4, 4), 1),         # cfg1: w = 128 too short (21.2 vs 22.3)
]


@pytest.mark.parametrize("cfg,best", SPLIT64_MEASURED)
def test_plan_simt_split64(L, cfg, best):
    from paper_2503_01253_b200 import nmspmm
    import torch
    p = nmspmm.nm_plan_query(*cfg, torch.float32)
    assert p["kernel"] == 1 and p["bm"] == 64, p
    assert p["split"] == best, p


# The bf16 slot kernel's geometry for nm_spmm (per-call prepack: m known) pinned to the choices the
# A-F study and the BASELINE timings support (profiles/r02e_protocol_summary.txt,
# profiles/r02g_protocol_af_after_retune.csv, profiles/r02g_sp_tmem_weights_ab.txt): bn = 128 H output
# columns per CTA, bm = NT tokens.
SLOT_GEOMETRY = [
    ((4096, 4096, 4096, 16, 32, 32), 256, 192),    # cfg2: H = 2 (50 %), 352 tiles
    ((2048, 11008, 4096, 12, 32, 32), 256, 208),   # cfg3 62.5 %: H = 2 (109 vs 124 us); 430 tiles
    ((256, 22016, 8192, 4, 32, 32), 128, 256),     # cfg4 m = 256: H = 1, one token tile
    ((2048, 11008, 4096, 8, 32, 32), 128, 256),    # cfg3 75 %: H = 1
    ((2048, 22016, 8192, 4, 32, 32), 128, 256),    # cfg4 87.5 %: H = 1
    ((2048, 4096, 4096, 12, 32, 32), 128, 256),    # A-F "E" 62.5 %: H = 2 would be < 2 waves -> H = 1
    ((1024, 2048, 2048, 16, 32, 32), 128, 128),    # A-F "D" 50 %: small grid -> H = 1, NT = 128
    ((512, 512, 512, 32, 32, 32), 128, 128),       # N = M, small grid: H = 1 (A-F 'A' at 0 %: 19.5 vs 15.9 TF)
    ((4096, 4096, 4096, 32, 32, 32), 256, 192),    # N = M, 4096^3: H = 2 (352 tiles)
]


@pytest.mark.parametrize("cfg,bn,bm", SLOT_GEOMETRY)
def test_plan_slot_geometry(L, cfg, bn, bm):
    from paper_2503_01253_b200 import nmspmm
    import torch
    p = nmspmm.nm_plan_query(*cfg, torch.bfloat16)
    assert p["kernel"] == 4
    assert (p["bn"], p["bm"]) == (bn, bm), p


@pytest.mark.parametrize("cfg,kid", [((1024, 1024, 1024, 8, 32, 4), 5),   # cfg5 L = 4: bf16 on the SIMT kernel
                                     ((256, 256, 256, 2, 4, 4), 5),      # cfg1 pattern
                                     ((64, 96, 192, 3, 8, 12), 5),       # L = 12
                                     ((64, 99, 192, 3, 8, 3), 0),        # L % 4 != 0: generic
                                     ((1024, 1024, 1024, 8, 32, 32), 4)])  # the slot kernel
def test_plan_bf16_fallback(L, cfg, kid):
    """bf16 shapes the slot kernel cannot take go to the fp32 SIMT kernel (exact fp32 copies),
    not the one-thread-per-element generic kernel, unless the SIMT kernel's shape rules fail."""
    from paper_2503_01253_b200 import nmspmm
    import torch
    assert nmspmm.nm_plan_query(*cfg, torch.bfloat16)["kernel"] == kid


# The SIMT row tile (nm_plan_query.bm, simt_row_tile) pinned to the faster of 64 / 128 measured on
# B200 (profiles/r02j_simt_row_tile.txt; the 128 column is the 128-row tile with its split rule).
ROW_TILE_MEASURED = [
    ((1024, 1024, 1024, 16, 32, 32), 64),    # 39.5 vs 47.1 us
    ((1024, 1024, 1024, 4, 32, 32), 64),     # 22.9 vs 27.9
    ((256, 13824, 5120, 4, 32, 32), 64),     # 114 vs 141
    ((2048, 1376, 4096, 8, 32, 32), 64),     # 173 vs 183 (cfg3-75 % 8-GPU shard)
    ((256, 256, 256, 2, 4, 4), 64),          # cfg1: 20.8 vs 27.2
    ((256, 22016, 8192, 4, 32, 32), 128),    # 258 vs 280
    ((2048, 2752, 8192, 4, 32, 32), 128),    # 303 vs 315 (cfg4-65B 8-GPU shard)
    ((2048, 2048, 2048, 16, 32, 32), 128),   # 188 vs 193
    ((4096, 4096, 4096, 16, 32, 32), 128),   # cfg2: 1208 vs 1200 (within 1 %)
    # the 100-point dataset (profiles/r02n_llama_dataset.csv 64-row vs r02e 128-row, fp32 8:32)
    ((256, 4096, 4096, 8, 32, 32), 128),     # 81.3 vs 86.4 (tiles64 128, w 1024: the split)
    ((256, 4096, 11008, 8, 32, 32), 128),    # 167 vs 209
    ((256, 8192, 8192, 8, 32, 32), 128),     # 219 vs 228
    ((4096, 512, 4096, 16, 32, 32), 128),    # cfg2 8-GPU shard: 220 vs 225
    ((256, 12288, 4096, 8, 32, 32), 64),     # 162 vs 203 (tiles64 384)
    ((512, 6656, 6656, 8, 32, 32), 64),      # 254 vs 322 (tiles64 416)
]


@pytest.mark.parametrize("cfg,bm", ROW_TILE_MEASURED)
def test_plan_simt_row_tile(L, cfg, bm):
    from paper_2503_01253_b200 import nmspmm
    import torch
    p = nmspmm.nm_plan_query(*cfg, torch.float32)
    assert p["kernel"] == 1 and p["bm"] == bm and p["threads"] == 2 * bm, p
