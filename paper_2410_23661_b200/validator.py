"""Python API over the C ABI (include/picker.h).

``Picker`` owns one library context on one CUDA device.  Tensors are used only
as device memory and streams; the calls marshal pointers and sizes.
"""
from __future__ import annotations

import ctypes
import json

import numpy as np
import torch

from . import _lib
from ._lib import PickerError, lib, picker_batch_t, picker_model_out_t, picker_model_params_t

NUM_COUNTS = 16
CODE_NAMES = {0: "IDEM_CHECKED", 1: "IDEM_KERNEL", 2: "NI_KERNEL_SO", 3: "NI_KERNEL_ATOMIC",
              4: "NI_KERNEL_IF", 5: "NI_KERNEL_PE", 6: "NI_KERNEL_NA", 7: "NI_PRECOND",
              8: "NI_GLOBAL", 9: "NI_OPAQUE", 10: "NI_OVERLAP", 11: "EXACT_SKIPPED",
              0xFE: "ERR_ARITY", 0xFF: "ERR_KERNEL"}
PATH_NAMES = {0: "shortcut", 1: "generic", 2: "jit", 3: "wide"}


def summary_text(summary) -> bytes:
    if isinstance(summary, (bytes, bytearray)):
        return bytes(summary)
    if isinstance(summary, str):
        return summary.encode()
    return json.dumps(summary, separators=(",", ":")).encode()


def verify_summaries(summary):
    """Parse + verify without a device.  Returns (status_or_count, message)."""
    t = summary_text(summary)
    buf = ctypes.create_string_buffer(1024)
    r = lib.picker_verify_summaries(t, len(t), buf, len(buf))
    return r, buf.value.decode()


def compile_summaries(summary, want_source=False):
    """Generate + NVRTC-compile the specialised module without a device.
    Returns (n_functions_or_status, message, source)."""
    t = summary_text(summary)
    msg = ctypes.create_string_buffer(8192)
    src = ctypes.create_string_buffer(1 << 24) if want_source else None
    r = lib.picker_compile_summaries(t, len(t), msg, len(msg), src, len(src) if src is not None else 0)
    return r, msg.value.decode(), (src.value.decode() if src is not None else None)


def records_tensor(rec, device=None):
    """numpy structured records (tracegen.records.REC_DTYPE) or a uint8 tensor -> u8[n, 32]."""
    if isinstance(rec, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(rec).view(np.uint8).reshape(-1, 32))
    else:
        t = rec
    return t.to(device) if device is not None else t


def _stream_handle(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _models_dict(out):
    return {"n": out.n, "n_idem": out.n_idem, "ckpt_bytes_all": out.ckpt_bytes_all,
            "ckpt_bytes_ni": out.ckpt_bytes_ni, "unknown_input": out.unknown_input,
            "preempt_ns_without": out.preempt_ns_without, "preempt_ns_with": out.preempt_ns_with,
            "hist_without": list(out.hist_without), "hist_with": list(out.hist_with)}


class Picker:
    """A validator context on one device (picker_create / picker_destroy)."""

    def __init__(self, device=None, **options):
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        h = ctypes.c_void_p()
        r = lib.picker_create(ctypes.byref(h), self.device.index or 0)
        if r != 0:
            raise PickerError(r, lib.picker_last_error(None).decode())
        self._h = h
        for k, v in options.items():
            self.set_option(k, v)
        self.n_kernels = 0

    def close(self):
        if getattr(self, "_h", None):
            lib.picker_destroy(self._h)
            self._h = None

    __del__ = close

    def _check(self, r):
        if r < 0:
            raise PickerError(r, lib.picker_last_error(self._h).decode())
        return r

    def set_option(self, key, value):
        self._check(lib.picker_set_option(self._h, key.encode(), int(value)))

    def load(self, summary):
        t = summary_text(summary)
        self.n_kernels = self._check(lib.picker_load_summaries(self._h, t, len(t)))
        return self.n_kernels

    def kernel_paths(self):
        n = self._check(lib.picker_kernel_info(self._h, None, None, 0))
        ids = (ctypes.c_uint32 * max(n, 1))()
        paths = (ctypes.c_uint8 * max(n, 1))()
        self._check(lib.picker_kernel_info(self._h, ids, paths, n))
        return {int(ids[i]): PATH_NAMES[int(paths[i])] for i in range(n)}

    def last_launch_count(self):
        return lib.picker_last_launch_count(self._h)

    @staticmethod
    def _batch(rec, args, packed):
        b = picker_batch_t()
        b.rec = rec.data_ptr() if rec.numel() else None
        b.args = args.data_ptr() if args.numel() else None
        b.args_len = args.numel()
        b.args_packed = 1 if packed else 0
        return b

    def validate(self, rec, args, *, packed=True, bits=True, counts=True, out=None, stream=None):
        """Validate device-resident records.  rec: u8[n,32] cuda tensor (or numpy
        records, copied to the device); args: int64 cuda tensor.  Returns
        (flags u8[n], bits i32[ceil(n/32)] or None, counts i64[16] or None) on the
        device; the work is queued on ``stream`` (default: current stream)."""
        rec = records_tensor(rec, self.device)
        if not torch.is_tensor(args):
            args = torch.from_numpy(np.asarray(args, dtype=np.int64))
        args = args.to(self.device)
        n = rec.shape[0]
        if out is None:
            flags = torch.empty(n, dtype=torch.uint8, device=self.device)
            bw = torch.empty((n + 31) // 32, dtype=torch.int32, device=self.device) if bits else None
            cnt = torch.empty(NUM_COUNTS, dtype=torch.int64, device=self.device) if counts else None
        else:
            flags, bw, cnt = out
        b = self._batch(rec, args, packed)
        self._check(lib.picker_validate_batch(
            self._h, ctypes.byref(b), n, flags.data_ptr(),
            bw.data_ptr() if bw is not None else None,
            cnt.data_ptr() if cnt is not None else None, _stream_handle(stream)))
        return flags, bw, cnt

    def validate_host(self, rec, args, *, packed=True, bits=True, counts=True, out=None,
                      stream=None):
        """End-to-end call with HOST buffers (pinned CPU tensors are fastest):
        H2D copy, validation and D2H copy inside the library.  Synchronous."""
        if isinstance(rec, np.ndarray):
            rec = records_tensor(rec)
        if not torch.is_tensor(args):
            args = torch.from_numpy(np.asarray(args, dtype=np.int64))
        n = rec.shape[0]
        if out is None:
            flags = torch.empty(n, dtype=torch.uint8)
            bw = torch.empty((n + 31) // 32, dtype=torch.int32) if bits else None
            cnt = torch.empty(NUM_COUNTS, dtype=torch.int64) if counts else None
        else:
            flags, bw, cnt = out
        b = self._batch(rec, args, packed)
        self._check(lib.picker_validate_batch_host(
            self._h, ctypes.byref(b), n, flags.data_ptr(),
            bw.data_ptr() if bw is not None else None,
            cnt.data_ptr() if cnt is not None else None, _stream_handle(stream)))
        return flags, bw, cnt

    def validate_sequence(self, rec, args, window, *, concurrent=False, stream=None):
        """Multi-kernel idempotency of consecutive windows of ``window`` launches
        (sequential list, or concurrent set).  Returns u8[ceil(n/window)] codes."""
        rec = records_tensor(rec, self.device)
        if not torch.is_tensor(args):
            args = torch.from_numpy(np.asarray(args, dtype=np.int64))
        args = args.to(self.device)
        n = rec.shape[0]
        out = torch.empty((n + window - 1) // window, dtype=torch.uint8, device=self.device)
        b = self._batch(rec, args, True)
        self._check(lib.picker_validate_sequence(self._h, ctypes.byref(b), n, int(window),
                                                 1 if concurrent else 0, out.data_ptr(),
                                                 _stream_handle(stream)))
        return out

    def exact_check(self, rec, args, *, max_points=1 << 20, counts=True, stream=None):
        """Exact (enumerating) verdicts for device-resident records (Fig. 3 strawman)."""
        rec = records_tensor(rec, self.device)
        if not torch.is_tensor(args):
            args = torch.from_numpy(np.asarray(args, dtype=np.int64))
        args = args.to(self.device)
        n = rec.shape[0]
        out = torch.empty(n, dtype=torch.uint8, device=self.device)
        cnt = torch.empty(NUM_COUNTS, dtype=torch.int64, device=self.device) if counts else None
        b = self._batch(rec, args, True)
        self._check(lib.picker_exact_check(
            self._h, ctypes.byref(b), n, out.data_ptr(),
            cnt.data_ptr() if cnt is not None else None, int(max_points),
            _stream_handle(stream)))
        return out, cnt

    def replicate(self, rec, args, ptr_mask, copies, *, first_copy=0, delta=1 << 37, stream=None):
        """K6 (picker_replicate): `copies` relocated copies of a device-resident
        trace, generated on the GPU.  rec: u8[n,32] / numpy records; args:
        int64; ptr_mask: bool per argument slot.  Returns (rec u8[n*copies,32],
        args int64[len(args)*copies]) on the device, queued on `stream`."""
        rec = records_tensor(rec, self.device)
        if not torch.is_tensor(args):
            args = torch.from_numpy(np.asarray(args, dtype=np.int64))
        args = args.to(self.device)
        mask = ptr_mask if torch.is_tensor(ptr_mask) else torch.from_numpy(np.asarray(ptr_mask, dtype=np.uint8))
        mask = mask.to(self.device, torch.uint8)
        n = rec.shape[0]
        rec_out = torch.empty((n * copies, 32), dtype=torch.uint8, device=self.device)
        args_out = torch.empty(args.numel() * copies, dtype=torch.int64, device=self.device)
        b = self._batch(rec, args, True)
        self._check(lib.picker_replicate(self._h, ctypes.byref(b), n, mask.data_ptr() if mask.numel() else None,
                                         int(copies), int(first_copy), int(delta), rec_out.data_ptr(),
                                         args_out.data_ptr() if args_out.numel() else None, _stream_handle(stream)))
        return rec_out, args_out

    def consumer_models(self, rec, args, codes, ctx_bytes=None, *, kill_ns=1000, save_bytes_per_us=1000,
                        stream=None):
        """Row f3 (picker_consumer_models): AR checkpoint bytes and Chimera
        preemption latency for a batch and its verdict codes.  Synchronous;
        returns a dict of Python ints (histograms as lists)."""
        rec = records_tensor(rec, self.device)
        if not torch.is_tensor(args):
            args = torch.from_numpy(np.asarray(args, dtype=np.int64))
        args = args.to(self.device)
        codes = codes.to(self.device) if torch.is_tensor(codes) else torch.from_numpy(
            np.asarray(codes, np.uint8)).to(self.device)
        n = rec.shape[0]
        cb = None
        if ctx_bytes is not None:
            cb = torch.from_numpy(np.asarray(ctx_bytes, np.uint64).view(np.int64)).to(self.device) \
                if not torch.is_tensor(ctx_bytes) else ctx_bytes.to(self.device)
        prm = picker_model_params_t(int(kill_ns), int(save_bytes_per_us))
        out = picker_model_out_t()
        b = self._batch(rec, args, True)
        self._check(lib.picker_consumer_models(
            self._h, ctypes.byref(b), n, codes.data_ptr(), cb.data_ptr() if cb is not None else None,
            ctypes.byref(prm), ctypes.byref(out), _stream_handle(stream)))
        return _models_dict(out)

    def validate_models(self, rec, args, ctx_bytes=None, *, kill_ns=1000, save_bytes_per_us=1000, out=None,
                        stream=None):
        """Verdicts and row f3 in one pass (picker_validate_models).  Synchronous;
        returns (flags, bits, counts) as ``validate`` plus the models dict of
        ``consumer_models``."""
        rec = records_tensor(rec, self.device)
        if not torch.is_tensor(args):
            args = torch.from_numpy(np.asarray(args, dtype=np.int64))
        args = args.to(self.device)
        n = rec.shape[0]
        if out is None:
            flags = torch.empty(n, dtype=torch.uint8, device=self.device)
            bw = torch.empty((n + 31) // 32, dtype=torch.int32, device=self.device)
            cnt = torch.empty(NUM_COUNTS, dtype=torch.int64, device=self.device)
        else:
            flags, bw, cnt = out
        cb = None
        if ctx_bytes is not None:
            cb = torch.from_numpy(np.asarray(ctx_bytes, np.uint64).view(np.int64)).to(self.device) \
                if not torch.is_tensor(ctx_bytes) else ctx_bytes.to(self.device)
        prm = picker_model_params_t(int(kill_ns), int(save_bytes_per_us))
        mo = picker_model_out_t()
        b = self._batch(rec, args, True)
        self._check(lib.picker_validate_models(
            self._h, ctypes.byref(b), n, flags.data_ptr(), bw.data_ptr() if bw is not None else None,
            cnt.data_ptr() if cnt is not None else None, cb.data_ptr() if cb is not None else None,
            ctypes.byref(prm), ctypes.byref(mo), _stream_handle(stream)))
        return (flags, bw, cnt), _models_dict(mo)
