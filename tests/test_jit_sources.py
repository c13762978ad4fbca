"""The device headers the library compiles at run time (csrc/jit.cu: NVRTC,
sm_100a) compile on the host too -- NVRTC needs no GPU -- with the options
jit.cu passes, for the three specialised kernels (config 2's geometry and
tile plan), so a host-only include or construct added to stages_dev.cuh /
sor_resident_dev.cuh / lesb_common.cuh fails here rather than as a silent
fallback on the GPU box."""

import ctypes
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1504_02264_b200", "csrc")
HEADERS = ("lesb_common.cuh", "stages_dev.cuh", "sor_resident_dev.cuh")
OPTS = ("--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "--prec-div=true", "--prec-sqrt=true",
        "--ftz=false", "--include-path=/usr/local/cuda/include")


def _nvrtc():
    for name in ("libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    pytest.skip("libnvrtc.so.12 not available")


def _compile(src: str, expr: str) -> bytes:
    nv = _nvrtc()
    prog = ctypes.c_void_p()
    names = (ctypes.c_char_p * len(HEADERS))(*[h.encode() for h in HEADERS])
    texts = (ctypes.c_char_p * len(HEADERS))(*[open(os.path.join(CSRC, h), "rb").read() for h in HEADERS])
    assert nv.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"lesb_jit.cu", len(HEADERS), texts, names) == 0
    assert nv.nvrtcAddNameExpression(prog, expr.encode()) == 0
    opts = (ctypes.c_char_p * len(OPTS))(*[o.encode() for o in OPTS])
    rc = nv.nvrtcCompileProgram(prog, len(OPTS), opts)
    n = ctypes.c_size_t()
    nv.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value)
    nv.nvrtcGetProgramLog(prog, log)
    assert rc == 0, log.value.decode(errors="replace")[-3000:]
    lowered = ctypes.c_char_p()
    assert nv.nvrtcGetLoweredName(prog, expr.encode(), ctypes.byref(lowered)) == 0
    size = ctypes.c_size_t()
    nv.nvrtcGetCUBINSize(prog, ctypes.byref(size))
    nv.nvrtcDestroyProgram(ctypes.byref(prog))
    assert size.value > 0
    return lowered.value


GEO = "#define LESB_JIT 1\n#define LESB_JIT_IM 150\n#define LESB_JIT_JM 150\n#define LESB_JIT_KM 90\n"


@pytest.mark.parametrize("expr", ["lesb::k_velnw_bondv1<true>", "lesb::k_fused_rhs<true>", "lesb::k_fused_rhs<false>"])
def test_stage_kernels_compile(expr):
    assert _compile(GEO + "#define FUSED_MINB 10\n#include \"stages_dev.cuh\"\n", expr)


@pytest.mark.parametrize("expr", ["lesb::k_sor_resident<true, false>", "lesb::k_sor_resident<false, true>"])
def test_resident_kernel_compiles(expr):
    plan = dict(NI=10, NJ=14, TIM=15, TJM=11, KK=46, KT=45, FSTRIDE=690, BSTRIDE=400200, PAD00=26, PAD01=0,
                PAD10=0, PAD11=0)
    d = GEO + "".join(f"#define LESB_JIT_RES_{k} {v}\n" for k, v in plan.items())
    assert _compile(d + "#include \"sor_resident_dev.cuh\"\n", expr)
