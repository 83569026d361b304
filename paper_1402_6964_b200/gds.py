"""cuFile (GPUDirect Storage) reads for the device-mode ChunkReader.

Replaces, for file-backed runs, the host bounce the reference's reader implies (reference
``pkg/src/tsnmf/matio.py:134-156``: ``f.read`` into a Python bytes object per chunk): ``cuFileRead`` moves file
bytes straight into a device buffer.  On a box with the ``nvidia-fs`` driver and a GDS-capable file system the
transfer is a DMA from storage to HBM; elsewhere libcufile runs in its compatibility mode (POSIX reads through
its own pinned bounce buffers) with the same API and results.  The library is bound at run time with ctypes
(``libcufile.so.0`` ships with the CUDA toolkit); nothing here is linked into ``libtsnmf_b200.so``, so a box
without libcufile only loses this optional path (``available()`` is False and ``ChunkReader(gds=True)``
raises ``TsnmfError``).

``cuFileDriverOpen`` is probed once in a child process with a time limit before it is called in-process
(``usable()``): on this pool's B200 boxes (containers without ``nvidia-fs``) libcufile 1.14 logs "running in
compatible mode" and then never returns from the driver open, and a reader that hangs is worse than one that
says so.  There ``ChunkReader(gds=True)`` raises ``TsnmfError`` and the pinned-buffer path is the one to use.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
import threading

from .errors import TsnmfError

_CU_FILE_HANDLE_TYPE_OPAQUE_FD = 1  # cufile.h: CUfileFileHandleType


class _CUfileError(ctypes.Structure):  # cufile.h: CUfileError_t {CUfileOpError err; CUresult cu_err;}
    _fields_ = [("err", ctypes.c_int), ("cu_err", ctypes.c_int)]


class _HandleUnion(ctypes.Union):
    _fields_ = [("fd", ctypes.c_int), ("handle", ctypes.c_void_p)]


class _CUfileDescr(ctypes.Structure):  # cufile.h: CUfileDescr_t
    _fields_ = [("type", ctypes.c_int), ("handle", _HandleUnion), ("fs_ops", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None
_lib_error: str | None = None
_driver_open = False


def _load():
    global _lib, _lib_error
    with _lock:
        if _lib is not None or _lib_error is not None:
            return _lib
        names = [os.environ.get("TSNMF_CUFILE_LIB"), "libcufile.so.0", "libcufile.so",
                 "/usr/local/cuda/targets/x86_64-linux/lib/libcufile.so.0"]
        last = None
        for name in names:
            if not name:
                continue
            try:
                lib = ctypes.CDLL(name)
            except OSError as exc:
                last = exc
                continue
            lib.cuFileDriverOpen.restype = _CUfileError
            lib.cuFileDriverOpen.argtypes = []
            lib.cuFileHandleRegister.restype = _CUfileError
            lib.cuFileHandleRegister.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_CUfileDescr)]
            lib.cuFileHandleDeregister.restype = None
            lib.cuFileHandleDeregister.argtypes = [ctypes.c_void_p]
            lib.cuFileBufRegister.restype = _CUfileError
            lib.cuFileBufRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
            lib.cuFileBufDeregister.restype = _CUfileError
            lib.cuFileBufDeregister.argtypes = [ctypes.c_void_p]
            lib.cuFileRead.restype = ctypes.c_ssize_t
            lib.cuFileRead.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_longlong,
                                       ctypes.c_longlong]
            _lib = lib
            return _lib
        _lib_error = f"libcufile not found ({last})"
        return None


def available() -> bool:
    """True when libcufile can be loaded (the driver itself is opened by the first FileHandle)."""
    return _load() is not None


_usable: tuple[bool, str] | None = None

_PROBE = r"""
import ctypes, sys
class E(ctypes.Structure):
    _fields_ = [("err", ctypes.c_int), ("cu_err", ctypes.c_int)]
lib = ctypes.CDLL(sys.argv[1])
lib.cuFileDriverOpen.restype = E
e = lib.cuFileDriverOpen()
sys.exit(0 if e.err == 0 else 3)
"""


def usable(timeout: float | None = None) -> bool:
    """True when libcufile loads AND its driver opens within ``timeout`` seconds (default 20, or
    ``TSNMF_CUFILE_PROBE_S``) in a child process; the verdict is cached (and inherited by child processes
    through ``TSNMF_CUFILE_USABLE``).  ``usable_reason()`` says why not."""
    global _usable
    with _lock:
        if _usable is not None:
            return _usable[0]
    if not available():
        verdict = (False, _lib_error or "libcufile not found")
    elif os.environ.get("TSNMF_CUFILE_USABLE") in ("0", "1"):
        verdict = (os.environ["TSNMF_CUFILE_USABLE"] == "1", "TSNMF_CUFILE_USABLE")
    else:
        limit = timeout if timeout is not None else float(os.environ.get("TSNMF_CUFILE_PROBE_S", "20"))
        try:
            rc = subprocess.run([sys.executable, "-c", _PROBE, _lib._name], timeout=limit, stdout=subprocess.DEVNULL,
                                stderr=subprocess.DEVNULL).returncode
            verdict = (rc == 0, "" if rc == 0 else f"cuFileDriverOpen failed in the probe process (exit {rc})")
        except subprocess.TimeoutExpired:
            verdict = (False, f"cuFileDriverOpen did not return within {limit:.0f} s on this box")
        os.environ["TSNMF_CUFILE_USABLE"] = "1" if verdict[0] else "0"
    with _lock:
        _usable = verdict
    return verdict[0]


def usable_reason() -> str:
    usable()
    return _usable[1] if _usable else ""


def _check(err: _CUfileError, what: str) -> None:
    if err.err != 0:
        raise TsnmfError(f"cuFile: {what} failed (cufile error {err.err}, cuda error {err.cu_err})", stage="ingest")


def _open_driver(lib) -> None:
    global _driver_open
    with _lock:
        if not _driver_open:
            _check(lib.cuFileDriverOpen(), "cuFileDriverOpen")
            _driver_open = True


class FileHandle:
    """A file registered with cuFile; ``read_into`` fills a device tensor region from a file offset."""

    def __init__(self, path):
        lib = _load()
        if lib is None:
            raise TsnmfError(f"cuFile is not available: {_lib_error}", stage="ingest")
        if not usable():
            raise TsnmfError(f"cuFile is not usable here: {usable_reason()}", stage="ingest")
        _open_driver(lib)
        self._lib = lib
        self.direct = True
        try:  # O_DIRECT is what a DMA path needs; page-cache-only file systems (tmpfs, overlay) reject it
            self._fd = os.open(os.fspath(path), os.O_RDONLY | os.O_DIRECT)
        except OSError:
            self._fd = os.open(os.fspath(path), os.O_RDONLY)
            self.direct = False
        descr = _CUfileDescr()
        descr.type = _CU_FILE_HANDLE_TYPE_OPAQUE_FD
        descr.handle.fd = self._fd
        descr.fs_ops = None
        self._fh = ctypes.c_void_p()
        err = lib.cuFileHandleRegister(ctypes.byref(self._fh), ctypes.byref(descr))
        if err.err != 0 and self.direct:  # retry without O_DIRECT (compatibility mode reads through the page cache)
            os.close(self._fd)
            self._fd = os.open(os.fspath(path), os.O_RDONLY)
            self.direct = False
            descr.handle.fd = self._fd
            err = lib.cuFileHandleRegister(ctypes.byref(self._fh), ctypes.byref(descr))
        if err.err != 0:
            os.close(self._fd)
            self._fd = -1
            _check(err, "cuFileHandleRegister")

    def read_into(self, dev_ptr: int, nbytes: int, file_offset: int, dev_offset: int = 0) -> int:
        """Blocking read of ``nbytes`` at ``file_offset`` into device memory ``dev_ptr + dev_offset``; returns
        the bytes read (short at end of file).  The data is in device memory when the call returns."""
        done = 0
        while done < nbytes:
            got = self._lib.cuFileRead(self._fh, ctypes.c_void_p(dev_ptr), nbytes - done, file_offset + done,
                                       dev_offset + done)
            if got < 0:
                raise TsnmfError(f"cuFile: cuFileRead failed ({got}, errno {ctypes.get_errno()})", stage="ingest")
            if got == 0:
                break
            done += got
        return done

    def close(self) -> None:
        if self._fd >= 0:
            self._lib.cuFileHandleDeregister(self._fh)
            os.close(self._fd)
            self._fd = -1

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
