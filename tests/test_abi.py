"""The C ABI library (no GPU needed): loads, exports every declared symbol,
matches the header's struct layout, and validates parameters before any CUDA
call (QPIR_E_PARAM / QPIR_E_DIMENSION name the offending field)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qpir.h")


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__._load_builder().build()
    from paper_2510_03631_b200 import _lib
    return _lib


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(qpir_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert set(names) == set(L.EXPORTS)
    lib = ctypes.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", nm), n


def test_params_struct_layout_matches_header(L, tmp_path):
    """Compile a C probe against include/qpir.h and compare offsets with ctypes."""
    fields = [f[0] for f in L.qpir_params._fields_]
    prog = ['#include <stdio.h>', '#include <stddef.h>', '#include "qpir.h"', "int main(void){",
            'printf("%zu\\n", sizeof(qpir_params));']
    prog += [f'printf("%zu\\n", offsetof(qpir_params, {f}));' for f in fields]
    prog += ["return 0;}"]
    c = tmp_path / "probe.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(c)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert vals[0] == ctypes.sizeof(L.qpir_params)
    for f, off in zip(fields, vals[1:]):
        assert getattr(L.qpir_params, f).offset == off, f


def _params(L, **kw):
    p = dict(n_cells=1024, n_ch=16, rec_bytes=8, m=0, lwe_n=1024, log_q=32, log_p=8,
             reserved0=0, seed_A=1, row_begin=0, row_end=0, device=0, flags=0)
    p.update(kw)
    return L.qpir_params(**p)


@pytest.mark.parametrize("kw,code,field", [
    (dict(log_p=7), 1, "log_p"),
    (dict(log_q=64), 1, "log_q"),
    (dict(lwe_n=0), 1, "lwe_n"),
    (dict(n_cells=0), 2, "n_cells"),
    (dict(row_end=129), 2, "row_end"),
    (dict(row_begin=64, row_end=64), 2, "row_begin"),
    (dict(reserved0=3), 1, "reserved0"),
    (dict(flags=6), 1, "flags"),
])
def test_setup_validates_before_cuda(L, kw, code, field):
    with pytest.raises(L.QpirError) as ei:
        L.qpir_setup(_params(L, **kw))
    assert ei.value.code == code
    assert field in str(ei.value)
    assert field in L.qpir_last_error(None)


def test_records_len_checked(L):
    import numpy as np
    with pytest.raises(L.QpirError) as ei:
        L.qpir_setup(_params(L), np.zeros(17, np.uint8))
    assert ei.value.code == 2 and "records_len" in str(ei.value)


def test_null_ctx_calls_fail_cleanly(L):
    assert L._L.qpir_answer(None, None, 0, None, 0, None) == L.QPIR_E_STATE
    assert L._L.qpir_kernel_launches(None) == 0
    L.qpir_destroy(None)


def test_fastmod_constant_is_exact():
    """limb_split_kernel reduces query entries with Lemire's fastmod
    (a mod p = hi64((M * a mod 2^64) * p), M = floor((2^64 - 1) / p) + 1): check the
    identity the kernel relies on for every p the tests use and edge-case a."""
    import random
    rng = random.Random(5)
    for p in (2, 3, 7, 255, 256, 257, 65521, 65536, 65537, 2**24 - 3, 2**31 - 1,
              4294967291, 2**32 - 1):
        M = (2**64 - 1) // p + 1
        xs = [0, 1, p - 1, p, p + 1, 2**32 - 1, 2**32 - 2, (2**32 - 1) // p * p] + \
             [rng.getrandbits(32) for _ in range(2000)]
        for a in xs:
            a &= 2**32 - 1
            assert (((M * a) % 2**64) * p) >> 64 == a % p, (p, a)
