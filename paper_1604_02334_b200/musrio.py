"""muSR data file I/O through the native loader/writer.

Drop-in for the reference's ``load_musr_data`` / ``store_musr_data``
(``pkg/src/blk/io.py:109-212``): same text format, same datasets, same
exceptions and messages, same bytes on disk.  The parsing and formatting of
the histogram counts -- all of the work at C4 scale (2^28 bins, ~1.2 GB of
text) -- runs multi-threaded in ``libmusr_b200.so`` (``musr_file_load`` /
``musr_file_store``, csrc/musr_io.cpp); this module builds the datasets and
turns the library's error reports into the reference's exceptions.

Files the native reader does not handle byte-exactly (non-ASCII text, integers
beyond int64) are read by ``_load_python``, a line-by-line restatement of
io.py:143-212.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .musr import MusrDataset, MusrError
from .theory import TheoryBinding, TheoryError

__all__ = ["FormatError", "load_musr_data", "store_musr_data"]

IO_OS, IO_MALFORMED, IO_BEFORE_HEADER, IO_UNKNOWN_KEY, IO_MISSING, IO_NEGATIVE = 1, 2, 3, 4, 5, 6
IO_BAD_MAP, IO_EMPTY_HIST, IO_BAD_DT, IO_NO_BLOCKS, IO_UNSUPPORTED = 7, 8, 9, 10, 11


class FormatError(ValueError):
    """Malformed data file (io.py:28-29)."""


class IoError(C.Structure):
    _fields_ = [("code", C.c_int), ("line", C.c_int64), ("text_off", C.c_int64),
                ("text_len", C.c_int64), ("detector", C.c_int64), ("bin", C.c_int64),
                ("missing", C.c_char * 96)]


class DetectorInfo(C.Structure):
    _fields_ = [("index", C.c_int64), ("dt", C.c_double), ("t0_bin", C.c_int64),
                ("n0_slot", C.c_int64), ("nbkg_slot", C.c_int64), ("n_map", C.c_int64),
                ("n_func", C.c_int64), ("n_counts", C.c_int64)]


def _lib_io():
    lib = _lib.load()
    if not getattr(lib, "_musr_io_typed", False):
        lib.musr_file_load.restype = C.c_int
        lib.musr_file_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p),
                                       C.POINTER(IoError)]
        lib.musr_file_n_detectors.restype = C.c_int
        lib.musr_file_n_detectors.argtypes = [C.c_void_p]
        lib.musr_file_detector.restype = C.c_int
        lib.musr_file_detector.argtypes = [C.c_void_p, C.c_int, C.POINTER(DetectorInfo)]
        lib.musr_file_copy.restype = C.c_int
        lib.musr_file_copy.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        lib.musr_file_free.restype = None
        lib.musr_file_free.argtypes = [C.c_void_p]
        lib.musr_file_store.restype = C.c_int
        lib.musr_file_store.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_char_p),
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_int,
                                        C.POINTER(IoError)]
        lib._musr_io_typed = True
    return lib


def _line_text(path, err: IoError) -> str:
    with open(path, "rb") as fh:
        fh.seek(err.text_off)
        return fh.read(err.text_len).decode("ascii")


def _raise(path, err: IoError):
    code, d = err.code, err.detector
    if code == IO_OS:
        raise OSError(err.bin, os.strerror(err.bin), str(path))
    if code == IO_MALFORMED:
        raise FormatError(f"{path}:{err.line}: malformed line: {_line_text(path, err)!r}")
    if code == IO_BEFORE_HEADER:
        raise FormatError(f"{path}:{err.line}: data before any DETECTOR header")
    if code == IO_UNKNOWN_KEY:
        raise FormatError(f"{path}:{err.line}: unknown key {_line_text(path, err).split()[0]!r}")
    if code == IO_MISSING:
        raise FormatError(f"{path}: detector {d} is missing {err.missing.decode()}")
    if code == IO_NEGATIVE:
        raise FormatError(f"{path}: detector {d} has a negative count at bin {err.bin}")
    if code == IO_BAD_MAP:
        raise TheoryError("map entries must be non-negative integers")
    if code == IO_EMPTY_HIST:
        raise FormatError(f"{path}: {MusrError(f'detector {d}: empty histogram')}")
    if code == IO_BAD_DT:
        raise FormatError(f"{path}: {MusrError(f'detector {d}: dt must be positive')}")
    if code == IO_NO_BLOCKS:
        raise FormatError(f"{path}: no detector blocks found")
    raise RuntimeError(f"musr_file_load: unexpected error code {code}")


def load_musr_data(path, n_threads: int = 0, dataset_type=MusrDataset,
                   binding_type=TheoryBinding) -> List:
    """Read a muSR data file (io.py:143-212) with the native parser.

    ``dataset_type`` / ``binding_type`` build the datasets (default: this
    package's mirrors; pass the reference's ``MusrDataset`` / ``TheoryBinding``
    to get its objects).  Counts arrive as float64, like MusrDataset.counts."""
    lib = _lib_io()
    handle = C.c_void_p()
    err = IoError()
    rc = lib.musr_file_load(os.fsencode(path), int(n_threads), C.byref(handle), C.byref(err))
    if rc != _lib.MUSR_OK:
        if err.code == IO_UNSUPPORTED:
            return _load_python(path, dataset_type, binding_type)
        _raise(path, err)
    try:
        out = []
        info = DetectorInfo()
        for i in range(lib.musr_file_n_detectors(handle)):
            lib.musr_file_detector(handle, i, C.byref(info))
            m = np.empty(info.n_map, dtype=np.int64)
            f = np.empty(info.n_func, dtype=np.float64)
            counts = np.empty(info.n_counts, dtype=np.float64)
            lib.musr_file_copy(handle, i, m.ctypes.data, f.ctypes.data, counts.ctypes.data, None)
            ds = dataset_type(detector_index=int(info.index), counts=counts, dt=float(info.dt),
                              t0_bin=int(info.t0_bin),
                              binding=binding_type(map=tuple(int(x) for x in m),
                                                   function_values=tuple(float(x) for x in f)),
                              n0_slot=int(info.n0_slot), nbkg_slot=int(info.nbkg_slot))
            out.append(ds)
        return out
    finally:
        lib.musr_file_free(handle)


def _header(ds) -> bytes:
    """The reference's header lines of one detector (io.py:127-133)."""
    lines = [f"DETECTOR {ds.detector_index}", f"dt {ds.dt!r}", f"t0 {ds.t0_bin}",
             f"n0_slot {ds.n0_slot}", f"nbkg_slot {ds.nbkg_slot}",
             "map " + " ".join(str(m) for m in ds.binding.map),
             "func " + " ".join(repr(v) for v in ds.binding.function_values)]
    return ("\n".join(lines) + "\n").encode()


def store_musr_data(path, datasets: Sequence, n_threads: int = 0) -> None:
    """Write datasets in the muSR text format (io.py:124-140), byte-identical
    to the reference writer; counts are formatted by the native writer."""
    lib = _lib_io()
    n = len(datasets)
    headers = [_header(ds) for ds in datasets]
    counts = [np.ascontiguousarray(np.asarray(ds.counts), dtype=np.float64) for ds in datasets]
    hdr = (C.c_char_p * max(n, 1))(*headers)
    ptr = (C.c_void_p * max(n, 1))(*[c.ctypes.data for c in counts])
    lens = np.array([len(c) for c in counts] or [0], dtype=np.int64)
    err = IoError()
    rc = lib.musr_file_store(os.fsencode(path), n, hdr, ptr,
                             lens.ctypes.data_as(C.POINTER(C.c_int64)), int(n_threads),
                             C.byref(err))
    if rc != _lib.MUSR_OK:
        _raise(path, err)


def _load_python(path, dataset_type=MusrDataset, binding_type=TheoryBinding) -> List:
    """Line-by-line restatement of load_musr_data (io.py:143-212) for files
    outside the native reader's byte-exact subset."""
    datasets = []
    block = None

    def finish(block):
        missing = [k for k in ("dt", "t0", "n0_slot", "nbkg_slot", "map", "counts") if k not in block]
        if missing:
            raise FormatError(f"{path}: detector {block['index']} is missing {', '.join(missing)}")
        counts = block["counts"]
        for bin_no, c in enumerate(counts):
            if c < 0:
                raise FormatError(
                    f"{path}: detector {block['index']} has a negative count at bin {bin_no}")
        try:
            return dataset_type(detector_index=block["index"],
                                counts=np.asarray(counts, dtype=np.int64), dt=block["dt"],
                                t0_bin=block["t0"],
                                binding=binding_type(map=block["map"],
                                                     function_values=block.get("func", ())),
                                n0_slot=block["n0_slot"], nbkg_slot=block["nbkg_slot"])
        except MusrError as exc:
            raise FormatError(f"{path}: {exc}") from exc

    setters = {"dt": float, "t0": int, "n0_slot": int, "nbkg_slot": int}
    with open(path) as fh:
        for lineno, raw in enumerate(fh, 1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            key = parts[0]
            try:
                if key == "DETECTOR":
                    if block is not None:
                        datasets.append(finish(block))
                    block = {"index": int(parts[1])}
                elif block is None:
                    raise FormatError(f"{path}:{lineno}: data before any DETECTOR header")
                elif key in setters:
                    block[key] = setters[key](parts[1])
                elif key == "map":
                    block["map"] = tuple(int(v) for v in parts[1:])
                elif key == "func":
                    block["func"] = tuple(float(v) for v in parts[1:])
                elif key == "counts":
                    block["counts"] = [int(v) for v in parts[1:]]
                elif "counts" in block:
                    block["counts"].extend(int(v) for v in parts)
                else:
                    raise FormatError(f"{path}:{lineno}: unknown key {key!r}")
            except FormatError:
                raise
            except (ValueError, IndexError) as exc:
                raise FormatError(f"{path}:{lineno}: malformed line: {line!r}") from exc
    if block is not None:
        datasets.append(finish(block))
    if not datasets:
        raise FormatError(f"{path}: no detector blocks found")
    return datasets
