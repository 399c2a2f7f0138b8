"""CPU checks of the boundary: libpcmm.so builds for sm_100a, loads without a GPU,
and exports every symbol include/pcmm.h declares (no compute calls here)."""
import ctypes
import os
import re
import shutil

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pcmm.h")).read()
    return sorted(set(re.findall(r"PCMM_API\s+[\w\s\*]*?\b(pcmm_\w+)\s*\(", src)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_library_exports_every_declared_symbol():
    from paper_2504_14497_b200 import build, pcmm
    build.build()
    lib = ctypes.CDLL(build.LIB)
    names = _declared()
    assert len(names) >= 17
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(pcmm.EXPORTS)
    lib.pcmm_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.pcmm_version()


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")
def test_library_is_sm100a_only():
    import subprocess
    from paper_2504_14497_b200 import build
    build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2504_14497_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f


def test_byte_path_workspace_bounded():
    # the Cussen byte path builds its tables in k-chunks when they would not fit the 2 GiB budget:
    # every w <= 8 at the 512^3 config stays within it (all tables of 512^3 w = 8 would be ~21 GB)
    from paper_2504_14497_b200 import pcmm
    L = pcmm.load()
    for w in range(1, 9):
        assert L.pcmm_workspace_bytes(512, 512, 512, w, 1) <= 2 << 30, w
    assert L.pcmm_workspace_bytes(256, 256, 256, 4, 1) < 512 << 20      # the headline run is not chunked


def test_validation_without_gpu():
    # argument errors are detected on the host before any device work
    from paper_2504_14497_b200 import pcmm
    L = pcmm.load()
    assert L.pcmm_workspace_bytes(0, 4, 4, 4, 1) == 0
    assert L.pcmm_workspace_bytes(4, 4, 4, 9, 1) == 0
    assert L.pcmm_workspace_bytes(4, 4, 4, 4, 1) > 0
    assert L.pcmm_workspace_bytes_wide(4, 4, 4, 16, 1) > 0
    assert L.pcmm_workspace_bytes_wide(4, 4, 4, 17, 1) == 0
    assert L.pcmm_workspace_bytes_wide(16385, 4, 4, 16, 1) == 0
    L.pcmm_paillier_workspace_bytes.restype = ctypes.c_size_t
    assert L.pcmm_paillier_workspace_bytes(4, 4, 4, 4, 3072, 1) > 0
    assert L.pcmm_paillier_workspace_bytes(4, 4, 4, 4, 4096, 1) == 0
    assert L.pcmm_paillier_workspace_bytes(4, 4, 4, 9, 3072, 0) == 0
    rc = L.pcmm_mul_cussen(None, 0, 4, 4, 4, 0, 4, None, None, None, 0, None)
    assert rc == pcmm.PCMM_EDIM
    rc = L.pcmm_mul_cussen(None, 4, 4, 4, 4, 0, 4, None, None, None, 0, None)
    assert rc == pcmm.PCMM_EINVAL
    assert L.pcmm_last_error()


def test_validation_of_the_next_entry_points_without_gpu():
    # NEXT-1 / NEXT-2 / NEXT-4 entry points reject bad arguments on the host, before any device work
    from paper_2504_14497_b200 import pcmm
    L = pcmm.load()
    P = pcmm
    # wide path: dimensions, null pointers, w range
    assert L.pcmm_mul_cussen_wide(None, 0, 4, 4, 12, 0, 4, None, None, None, 0, None) == P.PCMM_EDIM
    assert L.pcmm_mul_cussen_wide(None, 4, 4, 4, 12, 0, 4, None, None, None, 0, None) == P.PCMM_EINVAL
    assert L.pcmm_mul_schoolbook_wide(None, 20000, 4, 4, 12, 0, None, None, None, 0, None) == P.PCMM_EDIM
    assert L.pcmm_mul_strassen_wide(None, 4, 4, 4, 12, 0, 4, None, None, None, 0, None) == P.PCMM_EINVAL
    # NEXT-2 contexts
    assert L.pcmm_enc_ctx_bytes() == 256 + 2 * 32 * 256 * 64
    assert L.pcmm_bsgs_ctx_bytes(0) == 0 and L.pcmm_bsgs_ctx_bytes(29) == 0
    assert L.pcmm_bsgs_ctx_bytes(20) == 256 + (2 << 20) * 12
    assert L.pcmm_enc_ctx_init(None, None, None) == P.PCMM_EINVAL
    assert L.pcmm_encrypt_ctx(None, None, None, -1, None, None) == P.PCMM_EINVAL
    assert L.pcmm_encrypt_ctx(None, None, None, 0, None, None) == P.PCMM_OK       # empty batch
    assert L.pcmm_bsgs_init(0, None, None) == P.PCMM_EINVAL
    assert L.pcmm_decrypt_bsgs(None, None, 20, None, 1, 5, 4, None, None, None) == P.PCMM_EINVAL   # hi < lo
    assert L.pcmm_decrypt_bsgs(None, None, 4, None, 1, 0, 1 << 40, None, None, None) == P.PCMM_EINVAL  # range
    assert L.pcmm_decrypt_bsgs(None, None, 20, None, 0, 0, 9, None, None, None) == P.PCMM_OK   # empty batch
    # NEXT-4 Paillier
    words = (ctypes.c_uint32 * 16)(*([3] + [0] * 15))
    assert L.pcmm_paillier_mul(2, None, 4, 4, 4, 4, 4, words, 512, None, None, None, 0, None) == P.PCMM_EINVAL
    assert L.pcmm_paillier_mul(1, None, 0, 4, 4, 4, 4, words, 512, None, None, None, 0, None) == P.PCMM_EDIM
    even = (ctypes.c_uint32 * 16)(*([4] + [0] * 15))
    p = ctypes.c_void_p(1 << 20)        # aligned, never dereferenced: validation fails first
    assert L.pcmm_paillier_mul(1, p, 4, 4, 4, 4, 4, even, 512, p, p, p, 0, None) == P.PCMM_EINVAL
    assert L.pcmm_paillier_mul(1, p, 4, 4, 4, 4, 4, words, 4096, p, p, p, 0, None) == P.PCMM_ENOTSUP
    assert L.pcmm_paillier_mul(1, p, 4, 4, 4, 4, 5, words, 512, p, p, p, 0, None) == P.PCMM_ENOTSUP


def test_encrypt_rejects_bad_public_keys_without_gpu():
    # pcmm_encrypt validates H on the host (y^2 = x^3 - 3x + b, coordinates < p) before any launch;
    # the expected verdicts come from tests/ecref.py (OpenSSL points, SEC 2 constants), not the library
    from paper_2504_14497_b200 import pcmm as P
    from tests import ecref
    L = P.load()
    p = ctypes.c_void_p(1 << 20)                       # aligned, never dereferenced: validation fails first
    good = ecref.mulG(123456789)

    def rc(pk, r=p, ct=p):
        buf = ctypes.create_string_buffer(bytes(pk), 64)
        return L.pcmm_encrypt(buf, p, r, 4, ct, None)

    bad_y = bytearray(good)
    bad_y[63] ^= 1                                     # off the curve
    assert rc(bad_y) == P.PCMM_ENOTONCURVE
    x = int.from_bytes(good[:32], "big")
    y = int.from_bytes(good[32:], "big")
    unreduced = x.to_bytes(32, "big") + (y + ecref.P).to_bytes(33, "big")[1:] if y + ecref.P < 2**256 else None
    if unreduced is not None:                          # y + p as a 256-bit value: same residue, not reduced
        assert rc(unreduced) == P.PCMM_ENOTONCURVE
    assert rc(bytes(64)) == P.PCMM_ENOTONCURVE         # the identity
    neg = x.to_bytes(32, "big") + (ecref.P - y).to_bytes(32, "big")    # -H is a valid key
    assert rc(neg, r=ctypes.c_void_p((1 << 20) + 4)) == P.PCMM_EINVAL  # passes the curve check, misaligned r
    assert rc(good, ct=ctypes.c_void_p((1 << 20) + 8)) == P.PCMM_EINVAL
    for k in (1, 2, 3, ecref.Q - 1, 2**200 + 7):       # on-curve keys reach the alignment check only
        assert rc(ecref.mulG(k), r=ctypes.c_void_p((1 << 20) + 1)) == P.PCMM_EINVAL
    # x with y^2 = x^3 - 3x + b having no root: shift x until off-curve with y kept
    assert rc((x ^ 1).to_bytes(32, "big") + good[32:]) == P.PCMM_ENOTONCURVE
