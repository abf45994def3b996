"""The C-ABI library loads without a GPU and exports every function the
public header declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "specmd_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(esim_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("esim_router_launch", "esim_replay_launch", "esim_run_host", "esim_softmax_launch",
                 "esim_topk_launch", "esim_ls_create", "esim_ls_run", "esim_ffn_experts", "esim_last_error",
                 "esim_trace_jsonl_parse", "esim_trace_check_finite", "esim_set_host_sum", "esim_miss_decide"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2602_03921_b200 import build
    lib = ctypes.CDLL(build.build())
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_sizes_match_the_header():
    from paper_2602_03921_b200 import _abi
    from paper_2602_03921_b200.records import REC_DTYPE
    assert ctypes.sizeof(_abi.EsimConfig) == 184
    assert ctypes.sizeof(_abi.EsimCounters) == 360
    assert ctypes.sizeof(_abi.EsimTraceDesc) == 64
    assert ctypes.sizeof(_abi.EsimRouterOut) == 17 * 8
    assert ctypes.sizeof(_abi.EsimMissQuery) == 48 and ctypes.sizeof(_abi.EsimMissDecision) == 16
    assert REC_DTYPE.itemsize == 64
    from paper_2602_03921_b200.layer_step import EsimLSParams, EsimLSResult
    assert ctypes.sizeof(EsimLSParams) == 9 * 4           # incl. weight_format, prec_mask
    assert ctypes.sizeof(EsimLSResult) == 4 * 8 + 9 * 8


def test_gemv_decode_rejects_bad_geometry_before_any_device_work():
    """esim_ffn_experts_gemv validates its arguments on the host (-1, no CUDA
    call): unknown bit width, I not a multiple of 64, H not a multiple of 128
    or above 8192, 0 or > 4 tokens per expert, npad below max_tok, unaligned
    slot stride; no executed experts is a no-op (0)."""
    from paper_2602_03921_b200 import build
    lib = ctypes.CDLL(build.build())
    f = lib.esim_ffn_experts_gemv
    vp, i32 = ctypes.c_void_p, ctypes.c_int32
    f.argtypes = [vp, ctypes.c_int64, i32, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, vp]
    ok = dict(sb=3 * 2048 * 1024 * 2, bits=16, n=8, npad=16, mt=1, I=1024, H=2048)

    def call(**kw):
        a = dict(ok, **kw)
        return f(None, a["sb"], a["bits"], None, None, None, None, None, a["n"], a["npad"], a["mt"], a["I"], a["H"],
                 None)

    assert call(n=0) == 0
    for bad in (dict(bits=3), dict(bits=1), dict(I=1000), dict(H=2112), dict(H=16384), dict(mt=0), dict(mt=5),
                dict(npad=2, mt=4), dict(sb=3 * 2048 * 1024 * 2 + 8)):
        assert call(**bad) == -1, bad
