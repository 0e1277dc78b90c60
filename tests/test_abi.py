"""The C-ABI library builds for sm_100a, loads on a CPU-only host and exports every symbol of include/mxmoe.h."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mxmoe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mxm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2505_05799_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = _declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_signatures_cover_header():
    from paper_2505_05799_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_host_only_calls_without_gpu():
    """Metadata calls are pure host code: sizes and storage bits without a device."""
    import paper_2505_05799_b200 as mx
    mx.load()
    assert mx.storage_bits_per_weight(mx.Scheme(2, 16, 128, -1, False), 2048) == 2.25
    assert mx.storage_bits_per_weight(mx.Scheme(3, 16, 128, -1, False), 2048) == 3.25
    cb, sb, zb, pb = mx.quant_sizes(mx.Scheme(4, 16, 128, -1, False), 256, 1024)
    assert (cb, sb, zb) == (256 * 1024, 256 * 8 * 2, 256 * 8 * 2)
    assert pb * 8 == 256 * 1024 * 4.25
    from oracle.pack import packed_size
    for s in [(2, 16, 64, False), (3, 16, 128, True), (8, 16, -1, False), (5, 5, 128, True), (8, 8, -1, True),
              (16, 16, -1, True)]:
        assert mx.quant_sizes(mx.Scheme(s[0], s[1], s[2], s[2] if s[1] != 16 else -1, s[3]), 384, 1024)[3] == \
            packed_size(s[0], s[1], s[2], s[3], 384, 1024)
