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
