"""ctypes binding of libsssd.so (include/sssd.h).

The library is REQUIRED: importing a compute entry point without it raises
immediately — there is no CPU fallback.  Build it with
``python -m paper_2411_05894_b200.buildlib`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSSD_LIB") or os.path.join(_HERE, "libsssd.so")  # override: A/B builds

SSSD_MAX_P = 8
SSSD_MAX_DEPTH = 32
SSSD_MAX_DRAFT = 256
SSSD_ROW_TOKENS = 15
SSSD_INDEX_MAX = 32768
SSSD_STATUS_OFFSET = 8  # int32 status word in every propose / merge workspace
SSSD_PHASE_LOOKUP, SSSD_PHASE_SCAN, SSSD_PHASE_FUSE, SSSD_PHASE_BEGIN = 1, 2, 4, 8  # sssd_propose_phase bits
E_WORKSPACE = -4

u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class Cfg(C.Structure):
    _fields_ = [
        ("P", C.c_int32), ("dec_len", C.c_int32), ("branch_len", C.c_int32),
        ("input_branch_len", C.c_int32), ("M", C.c_int32), ("T", C.c_int32),
        ("use_datastore", C.c_int32), ("use_input", C.c_int32), ("n_input_trees", C.c_int32),
        ("has_separator", C.c_int32), ("separator", C.c_uint32), ("disc_stride", C.c_int32),
        ("disc", vp), ("fusion", C.c_int32),
    ]


class Elem(C.Structure):
    _fields_ = [("off", C.c_uint32), ("orig", C.c_uint32), ("len_m", C.c_uint32), ("pad", C.c_uint32)]


class Ds(C.Structure):
    _fields_ = [("rows", vp), ("tokens", vp), ("n_tokens", C.c_uint64), ("rank_base", C.c_uint64),
                ("n_rows", C.c_uint64), ("bucket", vp), ("n_buckets", C.c_uint32),
                ("kix", vp), ("kix_mask", C.c_uint64), ("kix_kmax", C.c_uint32)]


class Seqs(C.Structure):
    _fields_ = [("seq", vp), ("seq_off", vp), ("seq_len", vp), ("B", C.c_int32), ("max_len", C.c_int32)]


class DraftOut(C.Structure):
    _fields_ = [("size", vp), ("tokens", vp), ("parents", vp), ("depths", vp), ("mask", vp),
                ("priority", vp), ("source", vp), ("pos", vp)]  # (last three optional: NULL = skip)


class InputIndex(C.Structure):
    _fields_ = [("keys", vp), ("off", vp), ("len", vp), ("pos_bits", C.c_int32)]


class LookupOut(C.Structure):
    _fields_ = [("ranges", vp), ("samples", vp), ("n_conts", vp), ("p_cut", vp)]


_SIGS = {
    "sssd_error_string": (C.c_char_p, [C.c_int]),
    "sssd_last_error": (C.c_char_p, []),
    "sssd_version": (C.c_int, []),
    "sssd_sa_build_workspace": (C.c_size_t, [C.c_uint64]),
    "sssd_sa_build": (C.c_int, [vp, C.c_uint64, vp, vp, C.c_size_t, vp]),
    "sssd_sa_build_ex": (C.c_int, [vp, C.c_uint64, vp, vp, C.c_size_t, vp, C.POINTER(C.c_int32)]),
    "sssd_rows_build": (C.c_int, [vp, C.c_uint64, vp, vp, vp]),
    "sssd_rows_sa64": (C.c_int, [vp, C.c_uint64, vp, vp]),
    "sssd_sa_check_workspace": (C.c_size_t, [C.c_uint64]),
    "sssd_sa_check": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, vp, C.c_size_t, vp, vp]),
    "sssd_bucket_build": (C.c_int, [vp, C.c_uint64, C.c_uint32, vp, vp]),
    "sssd_kix_count": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint32, vp, vp]),
    "sssd_kix_build": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint32, vp, C.c_uint64, vp]),
    "sssd_widen_u16": (C.c_int, [vp, vp, C.c_int64, vp]),
    "sssd_rmsnorm_bf16": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int32, C.c_float, vp]),
    "sssd_rope_kv_bf16": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_int32, C.c_int32, C.c_float, vp]),
    "sssd_swiglu_bf16": (C.c_int, [vp, vp, C.c_int64, C.c_int32, vp]),
    "sssd_argmax_f32": (C.c_int, [vp, C.c_int64, C.c_int32, vp, vp]),
    "sssd_propose_workspace": (C.c_size_t, [C.POINTER(Cfg), C.c_int32, C.c_int32]),
    "sssd_propose_phase": (C.c_int, [C.POINTER(Ds), C.POINTER(Seqs), C.POINTER(Cfg), C.POINTER(DraftOut),
                                     C.POINTER(LookupOut), vp, C.c_size_t, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_int32, vp]),
    "sssd_gather_tails": (C.c_int, [vp, C.c_int32, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp]),
    "sssd_propose": (C.c_int, [C.POINTER(Ds), C.POINTER(Seqs), C.POINTER(Cfg), C.POINTER(DraftOut),
                               C.POINTER(LookupOut), vp, C.c_size_t, vp]),
    "sssd_input_index_build": (C.c_int, [C.POINTER(Seqs), C.POINTER(InputIndex), vp, C.c_int32, vp]),
    "sssd_propose_ex": (C.c_int, [C.POINTER(Ds), C.POINTER(Seqs), C.POINTER(InputIndex), C.POINTER(Cfg),
                                  C.POINTER(DraftOut), C.POINTER(LookupOut), vp, C.c_size_t, vp,
                                  C.POINTER(C.c_float)]),
    "sssd_propose_profile": (C.c_int, [C.POINTER(Ds), C.POINTER(Seqs), C.POINTER(Cfg), C.POINTER(DraftOut),
                                       vp, C.c_size_t, vp, C.POINTER(C.c_float)]),
    "sssd_set_cycle_probe": (None, [vp]),
    "sssd_set_fusion_form": (None, [C.c_int]),
    "sssd_workspace_status": (C.c_int, [C.POINTER(Cfg), C.c_int32, C.c_int32, vp, C.c_int32,
                                        C.c_int64, vp]),
    "sssd_find_ranges": (C.c_int, [C.POINTER(Ds), vp, vp, vp, C.c_int32, vp, vp]),
    "sssd_ds_lookup_workspace": (C.c_size_t, [C.POINTER(Cfg), C.c_int32]),
    "sssd_ds_lookup": (C.c_int, [C.POINTER(Ds), C.POINTER(Seqs), C.POINTER(Cfg), vp, vp, vp, vp,
                                 C.POINTER(LookupOut), vp, C.c_size_t, vp]),
    "sssd_input_scan_workspace": (C.c_size_t, [C.c_int32, C.c_int32]),
    "sssd_input_scan": (C.c_int, [C.POINTER(Seqs), C.POINTER(Cfg), vp, vp, vp, C.c_size_t, vp]),
    "sssd_merge_workspace": (C.c_size_t, [C.POINTER(Cfg), C.c_int32, C.c_int64]),
    "sssd_merge": (C.c_int, [vp, vp, vp, vp, C.c_int64, vp, C.c_int32, C.POINTER(Cfg),
                             C.POINTER(DraftOut), vp, C.c_size_t, vp]),
    "sssd_shard_search": (C.c_int, [C.POINTER(Ds), C.POINTER(Seqs), C.POINTER(Cfg), vp, vp]),
    "sssd_shard_gather": (C.c_int, [C.POINTER(Ds), C.POINTER(Cfg), C.c_int32, vp, vp, vp]),
    "sssd_shard_gather_pos": (C.c_int, [C.POINTER(Ds), C.POINTER(Cfg), C.c_int32, vp, vp, vp]),
    "sssd_rows_from_pos": (C.c_int, [vp, C.c_uint64, vp, C.c_int64, vp, vp]),
    "sssd_propose_pre": (C.c_int, [C.POINTER(Ds), C.POINTER(Seqs), C.POINTER(Cfg), vp, vp, C.POINTER(DraftOut),
                                   C.POINTER(LookupOut), vp, C.c_size_t, vp]),
    "sssd_teacher_predict": (C.c_int, [vp, vp, C.c_int32, vp, vp, vp, vp, vp, C.c_int32, vp, vp]),
    "sssd_accept": (C.c_int, [vp, vp, vp, C.c_int32, vp, C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp,
                              vp]),
    "sssd_kv_compact": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp,
                                  vp, C.c_int32, vp]),
    "sssd_tree_attention_workspace": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "sssd_tree_attention": (C.c_int, [vp, vp, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_float, vp, vp, C.c_size_t, vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class SSSDError(RuntimeError):
    pass


def lib() -> C.CDLL:
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SSSDError(f"{LIB_PATH} is missing: build it with `python -m paper_2411_05894_b200.buildlib`"
                            " (the package has no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().sssd_last_error().decode()
        if rc == -1:
            raise ValueError(msg)
        raise SSSDError(f"{lib().sssd_error_string(rc).decode()}: {msg}")


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise SSSDError("no CUDA device: the SSSD path runs only on the GPU (no CPU fallback)")
    lib()
    return torch.device("cuda", torch.cuda.current_device())
