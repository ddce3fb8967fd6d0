"""CPU-side checks of the drop-in boundary: libgecc_b200.so loads without a GPU, exports
every symbol include/gecc_b200.h declares (which includes every entry point of the
reference's sm2batch.h), keeps the reference's enum values, and fails loudly -- no CPU
fallback -- when asked to compute without a device."""
import ctypes as C
import os
import re

import pytest

import paper_2501_03245_b200 as gecc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = open(os.path.join(ROOT, "include", "gecc_b200.h")).read()

# the reference's C interface (sm2batch.h:44-105)
REFERENCE_ENTRY_POINTS = ["sm2b_ctx_new", "sm2b_ctx_free", "sm2b_version", "sm2b_status_str",
                          "sm2b_ledger_read", "sm2b_ledger_reset", "sm2b_keygen", "sm2b_sign",
                          "sm2b_verify", "sm2b_ecdh", "sm2b_crossover_n", "sm2b_bench_run"]


def test_library_builds_and_exports_every_declared_symbol():
    lib = gecc.lib()
    declared = sorted(set(re.findall(r"\b((?:sm2b|gecc)_[a-z0-9_]+)\s*\(", HDR)))
    assert len(declared) >= 35
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    for n in REFERENCE_ENTRY_POINTS:
        assert n in declared and hasattr(lib, n)


def test_metadata_and_status_codes_match_reference():
    lib = gecc.lib()
    assert lib.sm2b_version() == b"1.0.0"                      # capi.cpp:111
    names = {0: b"ok", 1: b"invalid argument", 2: b"malformed input", 3: b"invalid peer point",
             4: b"degenerate result", 5: b"nonce retries exhausted",
             6: b"cost model has no crossover", 7: b"internal error"}
    for code, text in names.items():                             # capi.cpp:113-125
        assert lib.sm2b_status_str(code) == text
    assert lib.sm2b_status_str(99) == b"unknown status"
    for name, val in re.findall(r"(SM2B_[A-Z_]+)\s*=\s*(\d+)", HDR):
        assert gecc.STATUS[int(val)]                             # enum values 0..7 as sm2batch.h:27-36
    out = C.c_uint64(0)
    assert lib.sm2b_crossover_n(C.c_uint64(1), C.c_uint64(5), C.c_uint64(500), C.byref(out)) == 0
    assert out.value == 21                                       # PAPER.md:466, bench.cpp:65-70
    assert lib.sm2b_crossover_n(C.c_uint64(1), C.c_uint64(0), C.c_uint64(500), C.byref(out)) == 6
    assert lib.sm2b_crossover_n(C.c_uint64(1), C.c_uint64(5), C.c_uint64(500), None) == 1
    assert lib.sm2b_ledger_read(None, None) == 1                 # test_capi.cpp:56


def test_no_cpu_fallback():
    """Without a CUDA device the context cannot be created; nothing computes on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gecc.GeccError):
        gecc.Context(gecc.SECP256K1)
    lib = gecc.lib()
    lib.sm2b_ctx_new.restype = C.c_void_p
    assert lib.sm2b_ctx_new(1, 0) is None
    # NULL context is an argument error everywhere, never a silent success
    assert lib.sm2b_verify(None, 0, None, None, None, None) == 1
    assert lib.sm2b_keygen(None, 1, 0, None, None) == 1


def test_product_never_imports_the_oracle():
    """oracle/ is test infrastructure: nothing under the package may reference it."""
    pkg = os.path.join(ROOT, "paper_2501_03245_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt, fn
                assert "gecc_oracle" not in txt and "libgecc_ref" not in txt, fn


def test_sm2batch_h_is_a_drop_in(tmp_path):
    """include/sm2batch.h: a C consumer of the reference's header name compiles against it and
    sees the reference's enum values and struct layouts (sm2batch.h:27-36,51-56,89-96)."""
    import subprocess
    src = tmp_path / "use.c"
    src.write_text(r'''
#include <stddef.h>
#include <stdio.h>
#include <sm2batch.h>
int main(void) {
    sm2b_bench_report r;
    sm2b_op_counts c;
    sm2b_status (*verify)(sm2b_ctx*, size_t, const uint8_t*, const uint8_t*, const uint8_t*, uint8_t*) = sm2b_verify;
    sm2b_status (*sign)(sm2b_ctx*, size_t, const uint8_t*, const uint8_t*, uint64_t, uint8_t*, int32_t*) = sm2b_sign;
    sm2b_status (*keygen)(sm2b_ctx*, uint64_t, size_t, uint8_t*, uint8_t*) = sm2b_keygen;
    sm2b_status (*ecdh)(sm2b_ctx*, size_t, const uint8_t*, const uint8_t*, uint8_t*, int32_t*) = sm2b_ecdh;
    sm2b_ctx* (*mk)(uint32_t, uint32_t) = sm2b_ctx_new;
    (void)verify; (void)sign; (void)keygen; (void)ecdh; (void)mk; (void)r; (void)c;
    printf("%d %d %d %d %d %d %d %d\n", SM2B_OK, SM2B_ERROR_INVALID_ARGUMENT, SM2B_ERROR_MALFORMED_INPUT,
           SM2B_ERROR_INVALID_PEER, SM2B_ERROR_DEGENERATE, SM2B_ERROR_NONCE_EXHAUSTED, SM2B_ERROR_NO_CROSSOVER,
           SM2B_ERROR_INTERNAL);
    printf("%zu %zu %zu %zu %zu\n", sizeof(sm2b_op_counts), offsetof(sm2b_op_counts, modinv), sizeof(sm2b_bench_report),
           offsetof(sm2b_bench_report, ops), offsetof(sm2b_bench_report, equivalence_checked));
    printf("%s\n", sm2b_version());
    return 0;
}
''')
    exe = tmp_path / "use"
    lib = os.path.join(ROOT, "paper_2501_03245_b200", "lib")
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                           "-L" + lib, "-lgecc_b200", "-Wl,-rpath," + lib])
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    assert out[0] == "0 1 2 3 4 5 6 7"
    assert out[1] == "32 24 72 24 64"     # u64 x4; {u64, double, double, 4 x u64, u64, int + pad}
    assert out[2] == "1.0.0"
    # where the reference lies beside us: the same translation unit against ITS header and library
    ref_inc = "/root/reference/proj/include"
    ref_lib = os.path.join(ROOT, "oracle", "_ref")
    if os.path.exists(os.path.join(ref_inc, "sm2batch.h")) and os.path.exists(os.path.join(ref_lib, "libgecc_ref.so")):
        exe2 = tmp_path / "use_ref"
        subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I" + ref_inc, str(src), "-o", str(exe2),
                               "-L" + ref_lib, "-lgecc_ref", "-Wl,-rpath," + ref_lib])
        assert subprocess.run([str(exe2)], capture_output=True, text=True, check=True).stdout.split("\n") == out
