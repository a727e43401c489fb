"""CPU: host-side logic of the product package and the C-ABI boundary.

No CUDA device is needed: these cover the storage layer (reference KATs),
argument validation (DimensionError before any launch, reference
messages), and that libpb_b200.so loads and exports every entry point
include/pb_b200.h declares.
"""
import ctypes
import os
import re
import struct

import numpy as np
import pytest
import torch

from conftest import REPO
import paper_1704_02457_b200 as pb
from paper_1704_02457_b200 import _native, level3, pack
from paper_1704_02457_b200.matstore import element_offset, memsize_panel_matrix


def test_element_offset_and_memsize_kats():
    # reference tests/test_matstore.py:14-17, 42-47
    assert element_offset(6, 3, 4, 8) == 46
    assert element_offset(4, 0, 4, 8) == 32
    assert memsize_panel_matrix(4, 4) == 192
    assert memsize_panel_matrix(5, 3) == 320
    assert memsize_panel_matrix(64, 64) == 33280  # C1 item


def test_element_offset_injective_in_bounds():
    for m in range(1, 21):
        for n in range(1, 21):
            cn = -(-n // 4) * 4
            offs = {element_offset(i, j, 4, cn) for i in range(m) for j in range(n)}
            assert len(offs) == m * n
            assert max(offs) < -(-m // 4) * 4 * cn


def test_panel_batch_views_on_cpu_storage():
    nb, m, n = 3, 6, 5
    p = pb.allocate_panel_batch(nb, m, n, device="cpu", zero=True, layout="interleaved")
    assert p.layout == "interleaved"
    assert p.storage.shape == (nb, memsize_panel_matrix(m, n) // 8)
    assert p.data.shape == (nb, 8 * 8)
    assert p.diag_inv.shape == (nb, 5)
    assert p.panels().shape == (nb, 2, 8, 4)
    p.panels()[1, 1, 3, 2] = 7.0  # row 6, col 3
    assert float(p.data[1, element_offset(6, 3, 4, 8)]) == 7.0
    p.panels()[1, 1, 3, 1] = 5.0  # row 5, col 3
    assert p.get(1, 5, 3) == 5.0
    d = p.descriptor()
    assert (d.m, d.n, d.cn, d.batch, d.stride) == (m, n, 8, nb, p.storage.shape[1])
    assert d.dA - d.pA == 64 * 8
    one = pb.allocate_panel_batch(1, m, n, device="cpu")
    bd = one.descriptor(7)
    assert bd.batch == 7 and bd.stride == 0 and bd.dA_stride == 0
    with pytest.raises(pb.DimensionError):
        p.descriptor(7)


def test_split_layout_planes_and_item_storage():
    nb, m, n = 3, 6, 5
    p = pb.allocate_panel_batch(nb, m, n, device="cpu", zero=True)
    assert p.layout == "split"
    assert p.storage.shape == (nb, 8 * 8) and p.diag_storage.shape == (nb, 5)
    d = p.descriptor()
    assert (d.stride, d.dA_stride) == (64, 5)
    assert d.dA == p.diag_storage.data_ptr()
    p.set(2, 5, 4, 3.5)
    p.diag_inv[2, 4] = 0.25
    assert p.get(2, 5, 4) == 3.5
    with pytest.raises(pb.DimensionError):
        p.get(3, 0, 0)
    with pytest.raises(pb.DimensionError):
        p.set(0, 6, 0, 1.0)
    # assembled reference layout == an interleaved batch holding the same values
    q = pb.allocate_panel_batch(nb, m, n, device="cpu", zero=True, layout="interleaved")
    q.set(2, 5, 4, 3.5)
    q.diag_inv[2, 4] = 0.25
    assert torch.equal(p.item_storage(), q.item_storage())
    assert p.item_bytes(2).tobytes() == q.item_bytes(2).tobytes()
    # shard views share memory
    s = p.shard(1, 3)
    assert s.batch == 2 and s.get(1, 5, 4) == 3.5 and s.descriptor().pA == p.descriptor().pA + 64 * 8
    # n = 4 items are back to back: one 128-byte line each
    four = pb.allocate_panel_batch(5, 4, 4, device="cpu")
    assert four.descriptor().stride == 16 and four.descriptor().dA_stride == 4
    assert pb.memsize_split_batch(5, 4, 4) == (5 * 128, 5 * 32)
    assert pb.panel_data_elems(5, 3) == 32


def test_create_panel_batch_validation():
    with pytest.raises(pb.MemoryLayoutError, match="required"):
        pb.create_panel_batch(2, 4, 4, torch.zeros(40, dtype=torch.float64))
    buf = torch.zeros(100, dtype=torch.float64)
    q = pb.create_panel_batch(2, 4, 4, buf)
    assert q.storage.data_ptr() == buf.data_ptr()  # no copy, contents untouched
    assert q.layout == "interleaved"
    with pytest.raises(pb.MemoryLayoutError):
        pb.create_panel_batch(1, 4, 4, torch.zeros(100, dtype=torch.float32))
    # split: data plane + diag plane
    data, diag = torch.zeros(2 * 16, dtype=torch.float64), torch.zeros(8, dtype=torch.float64)
    s = pb.create_panel_batch(2, 4, 4, data, diag)
    assert s.layout == "split" and s.diag_storage.data_ptr() == diag.data_ptr()
    with pytest.raises(pb.MemoryLayoutError, match="diag plane"):
        pb.create_panel_batch(2, 4, 4, data, torch.zeros(7, dtype=torch.float64))
    with pytest.raises(pb.MemoryLayoutError, match="data plane"):
        pb.create_panel_batch(2, 4, 4, torch.zeros(31, dtype=torch.float64), diag)
    with pytest.raises(pb.MemoryLayoutError, match="aligned"):
        pb.create_panel_batch(1, 4, 4, torch.zeros(40, dtype=torch.float64)[1:17], diag)


def test_dense_vector_batch_kats():
    # reference matstore.py:261-285, tests/test_matstore.py (memsize_vector)
    assert pb.memsize_vector(0) == 0
    assert pb.memsize_vector(1) == 64
    assert pb.memsize_vector(8) == 64
    assert pb.memsize_vector(9) == 128
    with pytest.raises(pb.DimensionError):
        pb.memsize_vector(-1)
    v = pb.allocate_vector_batch(3, 5, device="cpu", zero=True)
    assert v.data.shape == (3, 8) and v.memsize == 64 and v.stride == 8
    v.set(2, 4, 1.5)
    assert v.get(2, 4) == 1.5
    with pytest.raises(pb.DimensionError):
        v.get(2, 5)
    assert v.to_array().shape == (3, 5)
    buf = torch.arange(24, dtype=torch.float64)
    w = pb.create_vector_batch(3, 5, buf)
    assert w.data.data_ptr() == buf.data_ptr() and w.get(1, 0) == 8.0  # one 64-byte slot per item
    with pytest.raises(pb.MemoryLayoutError, match="required"):
        pb.create_vector_batch(4, 5, buf)
    # diag_inv exposed as a vector batch view
    p = pb.allocate_panel_batch(2, 6, 4, device="cpu", zero=True)
    p.diag_inv[1, 3] = 2.0
    dv = p.diag_vector()
    assert dv.len == 4 and dv.get(1, 3) == 2.0


def test_level3_bounds_errors_before_launch():
    a = pb.allocate_panel_batch(2, 4, 4, device="cpu")
    with pytest.raises(pb.DimensionError, match="A window"):
        level3.gemm_nt(5, 4, 4, 1.0, a, a, 0.0, a, a)
    with pytest.raises(pb.DimensionError, match="negative"):
        level3.gemm_nt(-1, 4, 4, 1.0, a, a, 0.0, a, a)
    with pytest.raises(pb.DimensionError):
        level3.syrk_ln(4, 5, 1.0, a, a, 0.0, a, a)
    with pytest.raises(pb.DimensionError):
        level3.trsm_rltn(4, 5, 1.0, a, a, a)
    with pytest.raises(pb.DimensionError):
        level3.potrf_l(3, a, a, n=5)
    with pytest.raises(pb.DimensionError):
        pb.SubRef(a, -1, 0)
    with pytest.raises(ValueError, match="variant"):
        level3.trsm(2, 2, 1.0, a, a, a, "rltx")
    with pytest.raises(NotImplementedError):
        level3.trsm(2, 2, 1.0, a, a, a, "llnu")
    with pytest.raises(pb.DimensionError):
        level3.getrf_pivot(5, 4, a, a)
    w = pb.allocate_panel_batch(2, 8, 10, device="cpu")
    with pytest.raises(pb.DimensionError, match="diag_inv"):
        level3.potrf_l(6, w, w.ref(0, 3))  # diag_inv[3:9] exceeds min(8, 10)
    with pytest.raises(pb.DimensionError):
        level3.getrf_nopivot(4, 4, a.ref(1, 0), a)
    # valid windows on CPU storage: refuses loudly (no CPU fallback)
    with pytest.raises(RuntimeError, match="CUDA"):
        level3.gemm_nt(4, 4, 4, 1.0, a, a, 0.0, a, a)
    with pytest.raises(RuntimeError, match="CUDA"):
        level3.getrf_pivot(4, 4, a, a)


def _header_symbols():
    text = open(os.path.join(REPO, "include", "pb_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*|int64_t)\s*(pb_\w+)\(", text, re.M)))


def test_native_library_exports_header_surface():
    lib = _native.load()
    syms = _header_symbols()
    assert len(syms) == 20, syms
    assert set(syms) == set(_native.SIGNATURES)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.pb_version() == _native.ABI_VERSION == 2
    # argument validation needs no device: a bad size returns -position
    d = pb.allocate_panel_batch(1, 4, 4, device="cpu").descriptor()
    assert lib.pb_dgemm_nt(-1, 4, 4, 1.0, ctypes.byref(d), 0, 0, ctypes.byref(d), 0, 0, 0.0, ctypes.byref(d), 0, 0,
                           ctypes.byref(d), 0, 0, None) == -1
    assert b"negative" in lib.pb_last_error()
    assert lib.pb_dpotrf_l(4, 5, ctypes.byref(d), 0, 0, ctypes.byref(d), 0, 0, None, None, 0, None) == -2
    assert lib.pb_dpotrf_l_worksize(4, 5, ctypes.byref(d), 0, 0, ctypes.byref(d), 0, 0) == -2
    # workspace sizing (no device needed): direct kernels need none, blocked
    # windows need panel workspace, unaligned blocked windows an aligned copy
    big = pb.allocate_panel_batch(3, 300, 300, device="cpu").descriptor()
    assert lib.pb_dpotrf_l_worksize(4, 4, ctypes.byref(d), 0, 0, ctypes.byref(d), 0, 0) == 0
    assert lib.pb_dpotrf_l_worksize(128, 128, ctypes.byref(big), 0, 0, ctypes.byref(big), 0, 0) == 0
    w256 = lib.pb_dpotrf_l_worksize(256, 256, ctypes.byref(big), 0, 0, ctypes.byref(big), 0, 0)
    assert w256 >= 3 * 2 * 128 * 128 * 8  # W (128 x 128) + T (128 x 128) per item
    assert lib.pb_dpotrf_l_worksize(256, 256, ctypes.byref(big), 0, 0, ctypes.byref(big), 1, 0) >= w256 + 3 * 256 * 256 * 8
    tall = pb.allocate_panel_batch(2, 600, 200, device="cpu").descriptor()
    # tall windows up to 128 columns: square factor + solve of the rows below straight into D, no workspace
    assert lib.pb_dpotrf_l_worksize(600, 20, ctypes.byref(tall), 0, 0, ctypes.byref(tall), 0, 0) == 0
    # wider ones: the rows below the first panel (W) and the trailing block (T) go through workspace
    assert lib.pb_dpotrf_l_worksize(600, 200, ctypes.byref(tall), 0, 0, ctypes.byref(tall), 0,
                                    0) >= 2 * (496 * 104 + 496 * 96) * 8
    # a call with less workspace than the query reports is refused before any launch
    assert lib.pb_dpotrf_l(256, 256, ctypes.byref(big), 0, 0, ctypes.byref(big), 0, 0, ctypes.c_void_p(8), None, 0,
                           None) == -10
    assert b"workspace" in lib.pb_last_error()
    assert lib.pb_dtrmm_rlnn_worksize(4, 40, ctypes.byref(big), 0, 0, ctypes.byref(big), 0, 0, ctypes.byref(big), 0,
                                      0) > 0  # in place, n > 24
    assert lib.pb_dtrmm_rlnn_worksize(4, 8, ctypes.byref(big), 0, 0, ctypes.byref(big), 0, 0, ctypes.byref(big), 0,
                                      0) == 0
    assert lib.pb_dgemm_nt(4, 4, 4, 1.0, ctypes.byref(d), 1, 0, ctypes.byref(d), 0, 0, 0.0, ctypes.byref(d), 0, 0,
                           ctypes.byref(d), 0, 0, None) == -5
    assert lib.pb_dgetrf(4, 4, ctypes.byref(d), 0, 0, ctypes.byref(d), 0, 0, 1, None, 4, None, None) == -10
    assert b"ipiv" in lib.pb_last_error()
    assert lib.pb_launch_count(0) == 0


def test_product_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_1704_02457_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(root, f)).read()
                assert "oracle" not in txt.replace("oracle's", ""), f


def test_colbatch_roundtrip_host_side():
    arr = np.arange(2 * 3 * 4, dtype=np.float64).reshape(2, 3, 4)
    cb = pack.ColBatch.from_array(arr, device="cpu")
    assert cb.lda == 3 and cb.data.shape == (2, 12)
    assert float(cb.data[1, 0 + 2 * 3]) == arr[1, 0, 2]
    assert np.array_equal(cb.to_array().numpy(), arr)


def test_bench_csv_matches_reference_schema(tmp_path):
    """bench.py --csv writes the reference's sweep CSV (bench.py:436-462):
    header, sorted rows, 17 significant digits, parseable by its reader."""
    import sys
    sys.path.insert(0, REPO)
    import bench
    pts, _ = bench.config_points("c2")
    points = [{"ms": 1.0 + i, "items": 1000 * (i + 1), "gflops": 10.0 * (i + 1)} for i in range(len(pts))]
    path = tmp_path / "sweep.csv"
    bench.emit_csv(bench.csv_rows(points, pts), str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == "routine,impl,m,n,k,seconds,gflops"
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == len(pts)
    ms = [int(r[2]) for r in rows]
    assert ms == sorted(ms) and rows[0][0] == "potrf_l" and rows[0][1] == "b200"
    assert float(rows[0][5]) == (1.0 / 1e3) / 1000 and float(rows[-1][6]) == 70.0
    # extended sidecar: the same seven columns, then gpus, batch, GB/s, roofline
    for i, p in enumerate(points):
        p.update(gbs_alg=100.0 * (i + 1), roofline_gflops=1000.0, roofline_frac=0.01 * (i + 1))
    ext = tmp_path / "sweep_ext.csv"
    bench.emit_csv_ext(bench.csv_rows(points, pts), points, pts, 2, str(ext))
    el = ext.read_text().splitlines()
    assert el[0].startswith(lines[0] + ",gpus,batch,")
    assert [e.split(",")[:7] for e in el[1:]] == rows
    assert el[1].split(",")[7] == "2" and int(el[1].split(",")[8]) == points[0]["items"]


def test_fixture_formats_match_the_reference(tmp_path):
    """§8f row 3: the matrix / OCP text fixtures written by the REFERENCE's own
    writers (tests/golden/make_fixture_golden.py) read back bit-exactly and
    are reproduced byte for byte by this package's writers."""
    from paper_1704_02457_b200 import fixtures
    gold = os.path.join(REPO, "tests", "golden")
    ref = open(os.path.join(gold, "ref_matrix_fixture.txt")).read()
    mat = fixtures.read_fixture(os.path.join(gold, "ref_matrix_fixture.txt"), device="cpu")
    assert (mat.rows, mat.cols) == (5, 3)
    lines = ref.splitlines()[1:]
    for i, line in enumerate(lines):
        for j, tok in enumerate(line.split()):
            got = mat.storage[0, pb.element_offset(i, j, 4, mat.panel_length)].item()
            assert struct.pack("<d", got) == struct.pack("<d", float(tok))
    out = tmp_path / "m.txt"
    fixtures.write_fixture(out, mat)
    assert out.read_text() == ref
    # a window of a larger batch item, and failing-item dumps
    big = pb.allocate_panel_batch(3, 9, 7, device="cpu", zero=True)
    for b in range(3):
        big.storage[b, :] = float(b)
    paths = fixtures.dump_failures(tmp_path / "fail", big, [-1, 4, -1], ai=2, aj=3, m=5, n=3)
    assert len(paths) == 1 and paths[0].endswith("item_1.txt")
    assert open(paths[0]).read() == ref.splitlines()[0] + "\n" + "\n".join(["1 1 1"] * 5) + "\n"
    nx, nu, stages, P = fixtures.read_ocp_fixture(os.path.join(gold, "ref_ocp_fixture.txt"))
    assert (nx, nu, len(stages), P.shape) == (2, 1, 2, (2, 2))
    out2 = tmp_path / "ocp.txt"
    fixtures.write_ocp_fixture(out2, nx, nu, stages, P)
    assert out2.read_text() == open(os.path.join(gold, "ref_ocp_fixture.txt")).read()


def test_bench_flop_counts_follow_the_reference():
    """bench.Point.flops_item restates the reference's flop_count
    (pkg/src/panelblas/bench.py:85-105); KATs after its
    tests/test_bench.py:13-21, plus bench.split_bytes == the split-layout size."""
    import sys
    sys.path.insert(0, REPO)
    import bench
    f = lambda op, m, n, k: bench.Point(op, m, n, k, 1).flops_item  # noqa: E731
    assert f("gemm_nt", 100, 100, 100) == 2e6
    assert f("gemm_nn", 0, 5, 5) == 0.0
    assert f("potrf_l", 3, 3, 3) == 9.0
    assert f("syrk_ln", 4, 4, 3) == 4 * 5 * 3
    assert f("trsm_rltn", 6, 4, 0) == 6 * 16
    assert f("trmm_rlnn", 6, 4, 0) == 6 * 16
    assert f("syrk_potrf_ln", 4, 4, 3) == 4 * 5 * 3 + 64 / 3.0
    assert f("getrf", 3, 3, 0) == 18.0
    nx, nu, N, s = 32, 8, 50, 40
    assert f("riccati_fact", nx, nu, N) == N * (s * nx * nx + s * (s + 1) * nx + s ** 3 / 3.0)
    with pytest.raises(ValueError):
        bench.Point("nope", 1, 1, 1, 1)
    for m in range(0, 41):
        for n in range(0, 41, 3):
            assert bench.split_bytes(m, n) == sum(pb.memsize_split_batch(1, m, n))
    # every C2 point carries ~2^34 flops (BASELINE configs[1])
    pts, _ = bench.config_points("c2")
    assert [p.n for p in pts] == [4, 8, 16, 32, 64, 128, 256]
    for p in pts:
        assert abs(p.batch * p.flops_item / 2 ** 34 - 1) < 1e-3


def _run_bench(*args, env=None):
    import subprocess
    import sys
    e = dict(os.environ, **(env or {}))
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True,
                          text=True, timeout=240, env=e)


def test_bench_cli_reference_arm_and_exit_codes():
    """bench.py CLI in a subprocess, after the reference's test_bench.py:147-171:
    the reference arm (host cores only, bounded sample) prints ONE JSON line
    with the contract keys; non-zero ranks exit 0 silently; an unknown
    --config exits non-zero before any CUDA call."""
    import json
    r = _run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.05",
                   "--only", "potrf_l n=4,potrf_l n=8")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    r1 = _run_bench("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                    env={"RANK": "1", "WORLD_SIZE": "2"})
    assert r1.returncode == 0 and r1.stdout.strip() == ""
    rb = _run_bench("--config", "bogus")
    assert rb.returncode != 0 and "unknown config" in rb.stderr
