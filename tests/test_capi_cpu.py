"""CPU-side checks of the product boundary: the C-ABI library loads and
exports every symbol include/zen_b200.h declares, the ctypes mirror binds all
of them, and with no GPU the library refuses to run (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "zen_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zen_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["zen_partition_of", "zen_to_sparse", "zen_hierarchical_hash",
                     "zen_universe_create", "zen_hash_bitmap_encode", "zen_hash_bitmap_decode",
                     "zen_bp_create", "zen_bp_sync_dense", "zen_bp_sync_sparse", "zen_bp_traffic",
                     "zen_bp_connect", "zen_bp_ipc_handle"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    import paper_2309_13254_b200 as z
    assert os.path.exists(z.LIB_PATH), "run `make lib` (build()) first"
    lib = ctypes.CDLL(z.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) == set(z.EXPORTED)


def test_host_only_entry_points_without_gpu():
    import paper_2309_13254_b200 as z
    lib = z.load()
    assert lib.zen_abi_version() == 1
    # host-side seed math equals the oracle's restatement
    from oracle import COracle
    co = COracle()
    for m, s in [(1, 0), (2024, 7), (2**63 + 3, 99)]:
        assert lib.zen_derive_seed(m, s) == co.derive_seed(m, s)
    f = z.HashFamily.make_worker(777, 3, 8, 3)
    assert [f.partition_seed] + f.slot_seeds == co.family_seeds(777, 8, 3, worker=3)


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2309_13254_b200 as z
    lib = z.load()
    h = ctypes.c_void_p()
    rc = lib.zen_ctx_create(0, ctypes.byref(h))
    assert rc == 7  # ZEN_E_CUDA
    assert b"no CPU fallback" in lib.zen_last_error_message()


def test_compat_header_compiles():
    """The C++ drop-in (include/zen_b200/compat.hpp) and its test build here."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("no g++")
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-Wall", "-Wextra",
                        "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                        os.path.join(ROOT, "tests", "cpp", "compat_test.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


def test_host_formats_without_gpu():
    """Host-side byte layouts: the frame header through the C-ABI
    (zen_frame_header / zen_frame_parse need no device) and the .zspt writer,
    against the reference's bytes (tests/golden/wire.npz)."""
    import io
    import numpy as np
    from conftest import load_golden
    import paper_2309_13254_b200 as z
    from paper_2309_13254_b200 import _lib as L
    lib = z.load()
    g = load_golden("wire")
    for c, row in enumerate(g["meta"]):
        kind, bs, cb, m = (int(x) for x in row[:4])
        count, ib, vb = (int(x) for x in row[7:])
        payload = g[f"c{c}_payload"]
        f = L.WireFormatC(kind, bs, cb)
        info = L.MessageInfoC(m, count, ib, vb, payload.size)
        hdr = np.zeros(33, np.uint8)
        assert lib.zen_frame_header(ctypes.byref(f), ctypes.byref(info),
                                    hdr.ctypes.data_as(ctypes.c_void_p)) == 0
        np.testing.assert_array_equal(hdr, g[f"c{c}_framed"][:33])
        framed = g[f"c{c}_framed"]
        f2, i2 = L.WireFormatC(), L.MessageInfoC()
        assert lib.zen_frame_parse(framed.ctypes.data_as(ctypes.c_void_p), framed.size,
                                   ctypes.byref(f2), ctypes.byref(i2)) == 0
        assert (f2.kind, i2.count, i2.payload_bytes) == (kind, count, payload.size)
        assert lib.zen_frame_parse(framed.ctypes.data_as(ctypes.c_void_p), framed.size - 1,
                                   ctypes.byref(f2), ctypes.byref(i2)) == 4  # truncated
    t = z.SparseTensor(int(g["zspt_m"][0]), g["zspt_idx"], g["zspt_val"])
    buf = io.BytesIO()
    z.write_sparse(buf, t)
    np.testing.assert_array_equal(np.frombuffer(buf.getvalue(), np.uint8), g["zspt_bytes"])
    buf.seek(0)
    assert z.read_sparse(buf) == t
