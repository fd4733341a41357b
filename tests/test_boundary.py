"""CPU tests of the C-ABI boundary: the library loads, exports every symbol include/gesr.h
declares, and host-checkable argument errors are rejected before any launch (no GPU needed:
these paths return before touching CUDA)."""
import ctypes
import os
import subprocess

import pytest

from paper_2511_21095_b200 import binding as gb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(gb.LIB_PATH):
        subprocess.check_call(["make", "-C", ROOT, "-j4"])
    return gb.lib()


def test_exports_every_header_symbol(L):
    syms = gb.header_symbols()
    assert set(syms) >= {"gesr_kv_project", "gesr_tasa_score", "gesr_hma_count",
                         "gesr_tasa_workspace_bytes", "gesr_status_string", "gesr_last_error",
                         "gesr_version"}
    out = subprocess.check_output(["nm", "-D", "--defined-only", gb.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for s in syms:
        assert s in exported, s
        assert hasattr(L, s)
    # nothing but the ABI is exported (the static CUDA runtime is kept local)
    assert all(s.startswith("gesr_") for s in exported if not s.startswith("_"))


def test_library_is_sm100a(L):
    out = subprocess.check_output(["cuobjdump", "--list-elf", gb.LIB_PATH], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", gb.LIB_PATH], text=True)
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass   # tcgen05 + TMA + TMEM


def test_status_strings(L):
    assert gb.status_string(0) == "GESR_OK"
    assert gb.status_string(1) == "GESR_ERR_INVALID_ARG"
    assert gb.status_string(2) == "GESR_ERR_UNSUPPORTED"
    assert gb.status_string(3) == "GESR_ERR_CUDA"
    assert gb.status_string(4) == "GESR_ERR_WORKSPACE"
    assert L.gesr_version() >= 100


P = ctypes.c_void_p
FAKE = P(0x10000)          # 16-byte aligned, never dereferenced on the error paths
MIS = P(0x10008)           # misaligned


def kv(L, U=FAKE, total_L=10, D_in=64, Wk=FAKE, Wv=FAKE, bk=None, bv=None, H=2, d=64, act=1,
       K=FAKE, V=FAKE):
    return L.gesr_kv_project(U, total_L, D_in, Wk, Wv, bk, bv, H, d, act, K, V, None)


def kvg(L, E=FAKE, n_E=100, D_in=64, rows=FAKE, total_L=10, Wk=FAKE, Wv=FAKE, H=2, d=64, act=1,
        K=FAKE, V=FAKE):
    return L.gesr_kv_project_gather(E, n_E, D_in, rows, total_L, Wk, Wv, None, None, H, d, act,
                                    K, V, None)


def test_kv_project_gather_validation(L):
    """gesr_kv_project_gather rejects bad arguments before any launch (no GPU needed)."""
    assert kvg(L, n_E=0) == gb.GESR_ERR_INVALID_ARG
    assert "n_E" in L.gesr_last_error().decode()
    assert kvg(L, n_E=1 << 31) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, d=48) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, D_in=20) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, total_L=-1) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, rows=None) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, E=None) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, E=MIS) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, rows=P(0x10002)) == gb.GESR_ERR_INVALID_ARG
    assert kvg(L, total_L=0, rows=None) == gb.GESR_OK      # empty problem: valid no-op


def test_tasa_score_gather_validation(L):
    """gesr_tasa_score_gather: table size, rows alignment and the unsupported self-key flag
    are rejected before any launch."""
    def call(n_E=100, rows=FAKE, flags=0, total_C=10, B=2):
        return L.gesr_tasa_score_gather(FAKE, n_E, 64, rows, total_C, FAKE, FAKE, None, 1, FAKE,
                                        FAKE, FAKE, B, 20, 2, 64, 0.0, 0, flags, FAKE, 0, None,
                                        P(0x100000), 1 << 30, None)
    assert call(n_E=0) == gb.GESR_ERR_INVALID_ARG
    assert call(rows=None) == gb.GESR_ERR_INVALID_ARG
    assert call(rows=P(0x10002)) == gb.GESR_ERR_INVALID_ARG
    assert call(flags=1) == gb.GESR_ERR_UNSUPPORTED
    assert call(total_C=0, rows=None) == gb.GESR_OK


def test_kv_project_validation(L):
    assert kv(L, d=48) == gb.GESR_ERR_INVALID_ARG
    assert "d=48" in L.gesr_last_error().decode()
    assert kv(L, D_in=20) == gb.GESR_ERR_INVALID_ARG
    assert kv(L, H=0) == gb.GESR_ERR_INVALID_ARG
    assert kv(L, act=7) == gb.GESR_ERR_INVALID_ARG
    assert kv(L, total_L=-1) == gb.GESR_ERR_INVALID_ARG
    assert kv(L, U=None) == gb.GESR_ERR_INVALID_ARG
    assert kv(L, K=MIS) == gb.GESR_ERR_INVALID_ARG
    assert kv(L, total_L=0, U=None) == gb.GESR_OK     # empty problem: valid no-op


def tasa(L, T=FAKE, total_C=10, D_in=64, co=FAKE, Wq=FAKE, bq=None, act=1, K=FAKE, V=FAKE,
         so=FAKE, B=2, total_L=10, H=2, d=64, scale=0.0, splits=0, flags=0, O=FAKE, odt=0,
         lse=None, ws=FAKE, wsb=1 << 30):
    return L.gesr_tasa_score(T, total_C, D_in, co, Wq, bq, act, K, V, so, B, total_L, H, d,
                             scale, splits, flags, O, odt, lse, ws, wsb, None)


def test_tasa_validation(L):
    assert tasa(L, d=96) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, odt=5) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, B=-1) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, flags=gb.GESR_TASA_SELF_KEY) == gb.GESR_ERR_UNSUPPORTED
    assert tasa(L, flags=0x8) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, splits=4) == gb.GESR_ERR_UNSUPPORTED       # split-L needs d = 128
    assert tasa(L, splits=-1) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, splits=65, d=128) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, T=None) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, O=MIS) == gb.GESR_ERR_INVALID_ARG
    assert tasa(L, ws=P(0x10010)) == gb.GESR_ERR_INVALID_ARG   # workspace must be 256-aligned
    assert tasa(L, wsb=16) == gb.GESR_ERR_WORKSPACE
    assert tasa(L, total_C=0, T=None) == gb.GESR_OK
    assert tasa(L, B=0) == gb.GESR_OK


def test_tasa_self_validation(L):
    def self_(Ks=FAKE, Vs=FAKE, d=64):
        return L.gesr_tasa_score_self(FAKE, 10, 64, FAKE, FAKE, None, 1, FAKE, FAKE, FAKE, 2, 10,
                                      2, d, 0.0, 0, Ks, Vs, FAKE, 0, None, FAKE, 1 << 30, None)
    assert self_(Ks=None) == gb.GESR_ERR_INVALID_ARG
    assert self_(Vs=MIS) == gb.GESR_ERR_INVALID_ARG
    assert self_(d=96) == gb.GESR_ERR_INVALID_ARG


def test_workspace_size(L):
    n = gb.tasa_workspace_bytes(1024, 1024000, 4, 128)
    # units list + Q [H, total_C, d] bf16 + an lse scratch [total_C, H] fp32 (self-key merge)
    base = 1024000 * 4 * 128 * 2 + 1024000 * 4 * 4
    assert n >= base and n < base + (1 << 20)
    assert gb.tasa_workspace_bytes(-1, 10, 4, 128) == 0
    assert gb.tasa_workspace_bytes(1, 10, 4, 100) == 0
    # split-L partials: [s, C, H] (m, l) + [s, C, H, d] fp32 on top of the unsplit workspace
    base = gb.tasa_workspace_bytes(1, 512, 4, 128, 1)
    assert gb.tasa_workspace_bytes(1, 512, 4, 128, 8) >= base + 8 * 512 * 4 * 130 * 4
    assert gb.tasa_workspace_bytes(1, 512, 4, 128, 0) >= base + 16 * 512 * 4 * 130 * 4  # auto bound
    assert gb.tasa_workspace_bytes(1, 512, 4, 128, 65) == 0


def hma(L, ui=FAKE, uo=FAKE, ii=FAKE, io=FAKE, co=FAKE, B=2, C=5, F=3, cap=0, counts=FAKE):
    return L.gesr_hma_count(ui, uo, ii, io, co, B, C, F, cap, counts, None)


def test_hma_validation(L):
    assert hma(L, F=-1) == gb.GESR_ERR_INVALID_ARG
    assert hma(L, F=300) == gb.GESR_ERR_INVALID_ARG
    assert hma(L, uo=None) == gb.GESR_ERR_INVALID_ARG
    assert hma(L, ii=P(0x10004)) == gb.GESR_ERR_INVALID_ARG
    assert hma(L, counts=P(0x10002)) == gb.GESR_ERR_INVALID_ARG
    assert hma(L, F=0) == gb.GESR_OK
    assert hma(L, C=0) == gb.GESR_OK


def test_binding_rejects_cpu_tensors(L):
    import torch
    U = torch.zeros(4, 64, dtype=torch.bfloat16)
    with pytest.raises(gb.GesrError):
        gb.kv_project(U, U, U, 1, 64)


def test_hma_embed_validation(L):
    def emb(E=FAKE, M=16, D_h=8, out=FAKE):
        return L.gesr_hma_count_embed(FAKE, FAKE, FAKE, FAKE, FAKE, 2, 5, 3, M, FAKE, E, D_h, out,
                                      None)
    assert emb(E=None) == gb.GESR_ERR_INVALID_ARG
    assert emb(M=0) == gb.GESR_ERR_INVALID_ARG
    assert emb(D_h=12) == gb.GESR_ERR_INVALID_ARG
    assert emb(out=None) == gb.GESR_ERR_INVALID_ARG
    assert emb(out=MIS) == gb.GESR_ERR_INVALID_ARG



def test_stu_output_validation(L):
    def stu(T=FAKE, C=10, D_in=64, O=FAKE, odt=0, Wg=FAKE, bg=None, g=FAKE, b=FAKE, eps=1e-5,
            Wo=FAKE, bo=None, X=None, H=2, d=64, D_out=128, Y=FAKE, ws=FAKE, wsb=1 << 30):
        return L.gesr_stu_output(T, C, D_in, O, odt, Wg, bg, g, b, eps, Wo, bo, X, H, d, D_out,
                                 Y, ws, wsb, None)
    assert stu(d=48) == gb.GESR_ERR_INVALID_ARG
    assert stu(D_out=48) == gb.GESR_ERR_INVALID_ARG
    assert "D_out=48" in L.gesr_last_error().decode()
    assert stu(odt=3) == gb.GESR_ERR_INVALID_ARG
    assert stu(eps=-1.0) == gb.GESR_ERR_INVALID_ARG
    assert stu(eps=float("nan")) == gb.GESR_ERR_INVALID_ARG
    assert stu(C=-1) == gb.GESR_ERR_INVALID_ARG
    assert stu(g=None) == gb.GESR_ERR_INVALID_ARG
    assert stu(Wo=None) == gb.GESR_ERR_INVALID_ARG
    assert stu(X=MIS) == gb.GESR_ERR_INVALID_ARG
    assert stu(wsb=16) == gb.GESR_ERR_WORKSPACE
    assert stu(C=0, T=None) == gb.GESR_OK                # empty problem: valid no-op
    # G then the gated rows in place: total_C * H * d bf16, 1 KB granular
    assert gb.stu_workspace_bytes(1000, 4, 128) == (1000 * 512 * 2 + 1023) // 1024 * 1024
    assert gb.stu_workspace_bytes(10, 2, 48) == 0


def test_nro_cross_validation(L):
    def nro(Wq=FAKE, g=FAKE, j=2, d=64, splits=0, ws=FAKE, wsb=1 << 30, C=10, B=2):
        return L.gesr_nro_cross_score(FAKE, C, 64, FAKE, Wq, g, None, 1, FAKE, FAKE, FAKE, B, 10,
                                      j, d, 0.0, splits, FAKE, 0, None, ws, wsb, None)
    assert nro(g=None) == gb.GESR_ERR_INVALID_ARG
    assert nro(g=MIS) == gb.GESR_ERR_INVALID_ARG
    assert nro(j=0) == gb.GESR_ERR_INVALID_ARG
    assert nro(d=96) == gb.GESR_ERR_INVALID_ARG
    assert nro(splits=65) == gb.GESR_ERR_INVALID_ARG
    assert nro(wsb=64) == gb.GESR_ERR_WORKSPACE
    assert nro(C=0) == gb.GESR_OK
    # the tasa workspace (256-aligned) followed by the folded query weight [j*d, D_in] bf16
    t = (gb.tasa_workspace_bytes(2, 10, 2, 64) + 255) // 256 * 256
    assert gb.nro_workspace_bytes(2, 10, 2, 64, 64) == t + 2 * 64 * 64 * 2


def test_layer_norm_validation(L):
    def ln(X=FAKE, rows=10, D=64, g=FAKE, b=FAKE, eps=1e-5, Y=FAKE):
        return L.gesr_layer_norm(X, rows, D, g, b, eps, Y, None)
    assert ln(D=12) == gb.GESR_ERR_INVALID_ARG
    assert ln(rows=-1) == gb.GESR_ERR_INVALID_ARG
    assert ln(eps=-1.0) == gb.GESR_ERR_INVALID_ARG
    assert ln(g=None) == gb.GESR_ERR_INVALID_ARG
    assert ln(Y=MIS) == gb.GESR_ERR_INVALID_ARG
    assert ln(rows=0, X=None) == gb.GESR_OK


def test_ro_cross_validation(L):
    def ro(seeds=FAKE, i=2, d=64, odt=0, ws=FAKE, wsb=1 << 30, B=2):
        return L.gesr_ro_cross_score(seeds, None, i, 64, FAKE, None, 1, FAKE, FAKE, FAKE, B, 10, d,
                                     0.0, FAKE, odt, ws, wsb, None)
    assert ro(seeds=None) == gb.GESR_ERR_INVALID_ARG
    assert ro(i=0) == gb.GESR_ERR_INVALID_ARG
    assert ro(d=96) == gb.GESR_ERR_INVALID_ARG
    assert ro(odt=4) == gb.GESR_ERR_INVALID_ARG
    assert ro(wsb=64) == gb.GESR_ERR_WORKSPACE
    assert ro(B=0) == gb.GESR_OK
