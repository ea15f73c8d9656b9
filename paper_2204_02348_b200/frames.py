"""Frame sources (holopipe/frames.py:30-102) staged onto the GPU.

A float32 source is held by reference and re-read on every run (the
reference contract, holopipe/frames.py:40-47); uint16 sources are handed to
the CUDA kernels as uint16 (converted to float32 in registers, optionally
transposed, holopipe/frames.py:89-101) instead of being re-converted into a
float32 staging buffer.  Sources may be numpy arrays (copied host->device on
every run) or CUDA torch tensors (zero-copy).
"""

from __future__ import annotations

import os

import numpy as np

from .errors import ErrorCode, HoloError

SOURCE_NONE, SOURCE_FLOAT32, SOURCE_UINT16, SOURCE_FILE = 0, 1, 2, 3
CAL_NONE, CAL_INTENSITY, CAL_FIELD = 0, 1, 2


def _is_torch(x):
    return type(x).__module__.startswith("torch")


class FrameSource:
    def __init__(self):
        self.kind = SOURCE_NONE
        self.f32 = None
        self.u16 = None
        self.transpose = 0
        self._dev = None          # reusable device staging buffer
        self._pinned = None       # device copy frozen by freeze() (AutoAlign)
        self._reg = None          # (ptr, nbytes) of a pageable host source registered with the driver

    def set_float32(self, buffer):
        if buffer is None:
            raise HoloError(ErrorCode.NULLPOINTER, "frame buffer is null")
        if not _is_torch(buffer):
            buffer = np.asarray(buffer, dtype=np.float32)
        elif buffer.dtype != __import__("torch").float32:
            buffer = buffer.float()
        self._release_if_other(buffer)
        self.kind, self.f32, self.u16, self._pinned = SOURCE_FLOAT32, buffer, None, None

    def set_uint16(self, buffer, transpose_mode=0):
        if buffer is None:
            raise HoloError(ErrorCode.NULLPOINTER, "frame buffer is null")
        if not _is_torch(buffer):
            arr = np.asarray(buffer)
            buffer = arr if arr.dtype == np.uint16 else arr.astype(np.uint16)
        self._release_if_other(buffer)
        self.kind, self.u16, self.f32, self._pinned = SOURCE_UINT16, buffer, None, None
        self.transpose = 1 if transpose_mode else 0

    def set_from_file(self, path):
        if not path:
            raise HoloError(ErrorCode.NULLPOINTER, "filename is null")
        if not os.path.isfile(path):
            raise HoloError(ErrorCode.FILENOTFOUND, path)
        raw = np.fromfile(path, dtype="<u2")
        self._unregister()
        self.kind, self.u16, self.f32, self._pinned = SOURCE_FILE, raw, None, None
        self.transpose = 0

    def float_buffer(self):
        if self.kind == SOURCE_FLOAT32:
            return self.f32
        return None

    def format(self):
        return 0 if self.kind == SOURCE_FLOAT32 else 1

    def staged(self, frame_count, width, height, device):
        """Device tensor holding at least frame_count frames (flat), and its format.

        Returns (tensor, fmt, transpose).  Raises INVALIDDIMENSION for short
        buffers (holopipe/frames.py:85-87).
        """
        import torch
        need = frame_count * width * height
        if self.kind == SOURCE_NONE:
            raise HoloError(ErrorCode.NULLPOINTER, "no frame source set")
        src = self.f32 if self.kind == SOURCE_FLOAT32 else self.u16
        n = src.numel() if _is_torch(src) else src.size
        if n < need:
            raise HoloError(ErrorCode.INVALIDDIMENSION, f"frame buffer holds {n} pixels, need {need}")
        fmt = self.format()
        tr = self.transpose if fmt == 1 else 0
        if self._pinned is not None and self._pinned.numel() >= need:
            return self._pinned, fmt, tr
        if _is_torch(src):
            flat = src.reshape(-1)[:need]
            if flat.device != device:
                flat = flat.to(device)
            return flat.contiguous(), fmt, tr
        flat = np.ascontiguousarray(src.reshape(-1)[:need])
        host = torch.from_numpy(flat if fmt == 0 else flat.view(np.int16))
        dt = torch.float32 if fmt == 0 else torch.int16
        if self._dev is None or self._dev.numel() < need or self._dev.dtype != dt or self._dev.device != device:
            self._dev = torch.empty(need, dtype=dt, device=device)
        dev = self._dev[:need]
        dev.copy_(host)
        return dev, fmt, tr

    def host_array(self):
        """The host-resident source buffer (numpy or CPU tensor), or None for device sources."""
        src = self.f32 if self.kind == SOURCE_FLOAT32 else self.u16
        if src is None:
            return None
        if _is_torch(src):
            if src.device.type != "cpu":
                return None
            return src if src.is_contiguous() else None
        arr = np.asarray(src)
        if not arr.flags["C_CONTIGUOUS"]:
            return None
        if self.kind == SOURCE_FLOAT32 and arr.dtype != np.float32:
            return None
        return arr

    def ensure_registered(self):
        """Page-lock the current pageable host source in place (cudaHostRegister) so that the window
        uploads run at pinned-memory speed.  holopipe holds the caller's frame buffer by reference and
        re-reads it on every run (holopipe/frames.py:40-47), so the registration is made once per buffer
        and released when the source changes (or this object is collected).  A failed registration
        leaves the buffer pageable (correct, slower)."""
        arr = self.host_array()
        if arr is None or _is_torch(arr):
            return
        ptr, nbytes = arr.ctypes.data, arr.nbytes
        if self._reg == (ptr, nbytes) or getattr(self, "_tried", None) == (ptr, nbytes) or nbytes == 0:
            return
        self._unregister()
        from . import native
        self._tried = (ptr, nbytes)   # one attempt per buffer (an already page-locked range stays as it is)
        if native.lib().hpg_host_register(ptr, nbytes) == 0:
            self._reg = (ptr, nbytes)

    def _release_if_other(self, buffer):
        """Keep the registration when the same host buffer is set again (a caller re-arming its batch)."""
        if self._reg is None:
            return
        if not _is_torch(buffer) and isinstance(buffer, np.ndarray) and buffer.flags["C_CONTIGUOUS"] \
                and (buffer.ctypes.data, buffer.nbytes) == self._reg:
            return
        self._unregister()

    def _unregister(self):
        if self._reg is not None:
            from . import native
            native.lib().hpg_host_unregister(self._reg[0])
            self._reg = None

    def __del__(self):
        try:
            self._unregister()
        except Exception:
            pass

    def freeze(self, tensor):
        """Keep a device copy for repeated evaluations (no external mutation expected)."""
        self._pinned = tensor

    def thaw(self):
        self._pinned = None


class RefCalibration:
    """Reference-wave calibration state (holopipe/frames.py:105-187)."""

    def __init__(self):
        self.kind = CAL_NONE
        self.enabled = 0
        self.raw = None
        self.wavelength_count = 0

    def set_intensity(self, cal, wavelength_count, width, height):
        if cal is None or width <= 0 or height <= 0 or wavelength_count <= 0:
            self.enabled = 0
            return False
        self.kind = CAL_INTENSITY
        self.raw = np.asarray(cal).reshape(wavelength_count, height, width).astype(np.float32)
        self.wavelength_count = int(wavelength_count)
        self.enabled = 1
        return True

    def set_field(self, cal, wavelength_count, width, height):
        if cal is None or width <= 0 or height <= 0 or wavelength_count <= 0:
            self.enabled = 0
            return False
        self.kind = CAL_FIELD
        self.raw = np.asarray(cal, dtype=np.complex64).reshape(wavelength_count, height, width).copy()
        self.wavelength_count = int(wavelength_count)
        self.enabled = 1
        return True

    def set_from_file(self, path, wavelength_count, width, height):
        if not path:
            raise HoloError(ErrorCode.NULLPOINTER, "filename is null")
        if not os.path.isfile(path):
            raise HoloError(ErrorCode.FILENOTFOUND, path)
        if width <= 0 or height <= 0 or wavelength_count <= 0:
            self.enabled = 0
            return False
        count = wavelength_count * width * height
        size = os.path.getsize(path)
        if size == count * 2:
            return self.set_intensity(np.fromfile(path, dtype="<u2", count=count),
                                      wavelength_count, width, height)
        if size == count * 8:
            raw = np.fromfile(path, dtype="<f4", count=count * 2)
            return self.set_field((raw[0::2] + 1j * raw[1::2]).astype(np.complex64),
                                  wavelength_count, width, height)
        raise HoloError(ErrorCode.INVALIDARGUMENT, f"file size {size} matches no calibration layout")

    def disable(self):
        self.enabled = 0

    def normalised_intensity(self):
        if self.kind == CAL_INTENSITY:
            inten = self.raw.astype(np.float64)
        elif self.kind == CAL_FIELD:
            inten = np.abs(self.raw.astype(np.complex128)) ** 2
        else:
            return None
        peak = inten.max()
        return np.ones_like(inten) if peak <= 0 else inten / peak
