"""ctypes binding of libpicker.so (include/picker.h).  Argument marshalling only:
every step of the validation runs in the library's CUDA kernels.  There is no
CPU fallback: if the shared library is missing this module raises on import."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpicker.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2410_23661_b200.build` "
        "(or __graft_entry__.build()); there is no fallback path")

lib = ctypes.CDLL(LIB_PATH)


class picker_rec_t(ctypes.Structure):
    _fields_ = [("kernel_id", ctypes.c_uint32), ("nargs", ctypes.c_uint32),
                ("grid_x", ctypes.c_uint32), ("grid_y", ctypes.c_uint16),
                ("grid_z", ctypes.c_uint16), ("block_x", ctypes.c_uint16),
                ("block_y", ctypes.c_uint16), ("block_z", ctypes.c_uint16),
                ("reserved", ctypes.c_uint16), ("arg_off", ctypes.c_uint64)]


class picker_batch_t(ctypes.Structure):
    _fields_ = [("rec", ctypes.c_void_p), ("args", ctypes.c_void_p),
                ("args_len", ctypes.c_uint64), ("args_packed", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


assert ctypes.sizeof(picker_rec_t) == 32

MODEL_HIST = 129


class picker_model_params_t(ctypes.Structure):
    _fields_ = [("kill_ns", ctypes.c_uint64), ("save_bytes_per_us", ctypes.c_uint64)]


class picker_model_out_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("n_idem", ctypes.c_uint64), ("ckpt_bytes_all", ctypes.c_uint64),
                ("ckpt_bytes_ni", ctypes.c_uint64), ("unknown_input", ctypes.c_uint64),
                ("preempt_ns_without", ctypes.c_uint64), ("preempt_ns_with", ctypes.c_uint64),
                ("hist_without", ctypes.c_uint64 * MODEL_HIST), ("hist_with", ctypes.c_uint64 * MODEL_HIST)]

P = ctypes.c_void_p
U64 = ctypes.c_uint64

SIGNATURES = {
    "picker_create": (ctypes.c_int, [ctypes.POINTER(P), ctypes.c_int]),
    "picker_destroy": (None, [P]),
    "picker_last_error": (ctypes.c_char_p, [P]),
    "picker_load_summaries": (ctypes.c_int, [P, ctypes.c_char_p, ctypes.c_size_t]),
    "picker_verify_summaries": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p,
                                               ctypes.c_size_t]),
    "picker_compile_summaries": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p,
                                                ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]),
    "picker_validate_batch": (ctypes.c_int, [P, ctypes.POINTER(picker_batch_t), U64, P, P, P, P]),
    "picker_validate_batch_host": (ctypes.c_int, [P, ctypes.POINTER(picker_batch_t), U64, P, P, P,
                                                  P]),
    "picker_exact_check": (ctypes.c_int, [P, ctypes.POINTER(picker_batch_t), U64, P, P, U64, P]),
    "picker_replicate": (ctypes.c_int, [P, ctypes.POINTER(picker_batch_t), U64, P, U64, U64, ctypes.c_int64, P, P,
                                        P]),
    "picker_validate_sequence": (ctypes.c_int, [P, ctypes.POINTER(picker_batch_t), U64, ctypes.c_uint32,
                                                ctypes.c_uint32, P, P]),
    "picker_consumer_models": (ctypes.c_int, [P, ctypes.POINTER(picker_batch_t), U64, P, P,
                                              ctypes.POINTER(picker_model_params_t),
                                              ctypes.POINTER(picker_model_out_t), P]),
    "picker_validate_models": (ctypes.c_int, [P, ctypes.POINTER(picker_batch_t), U64, P, P, P, P,
                                              ctypes.POINTER(picker_model_params_t),
                                              ctypes.POINTER(picker_model_out_t), P]),
    "picker_kernel_info": (ctypes.c_int, [P, P, P, ctypes.c_uint32]),
    "picker_set_option": (ctypes.c_int, [P, ctypes.c_char_p, ctypes.c_int64]),
    "picker_last_launch_count": (ctypes.c_int, [P]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

STATUS = {0: "OK", -1: "EINVAL", -2: "EFORMAT", -3: "EUNSAFE", -4: "ENOTLOADED", -5: "ECUDA",
          -6: "ENOMEM"}


class PickerError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.msg = msg
