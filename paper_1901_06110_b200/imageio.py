"""PGM / PFM image files — drop-in for the file I/O of pnprestore/image.py
(read_image / write_image and the ImageFormatError family, image.py:16-31,
169-280).  Host-side byte parsing (it never touches the GPU):

* PGM: ASCII ``P2`` and binary ``P5``, maxval in (0, 65535], ``#`` comments
  between header tokens, big-endian 16-bit samples when maxval > 255;
  samples are scaled to [0, 1] by maxval.
* PFM: grayscale ``Pf`` only, float32, scanlines bottom-to-top, a negative
  scale meaning little-endian.
* write: ``pgm8`` (clamp to [0, 1], round half up to 8 bits, binary P5) or
  ``pfm`` (float32, little-endian, scale -1.0).
"""

from __future__ import annotations

import re

import numpy as np

from . import _arrays as A


class ImageFormatError(ValueError):
    """A file that is not a readable PGM / PFM image."""


class UnsupportedFormatError(ImageFormatError):
    """Magic number of a format this reader does not handle."""


class MalformedHeaderError(ImageFormatError):
    """Header fields missing, non-numeric or out of range."""


class TruncatedPayloadError(ImageFormatError):
    """Fewer samples than the header announces."""


_WS = b" \t\n\r\x0b\x0c"


def _header_tokens(buf: bytes, count: int) -> tuple[list[bytes], int]:
    """``count`` whitespace-separated tokens after the 2-byte magic, with
    '#'-to-end-of-line comments skipped; returns them and the offset just past
    the single whitespace byte that ends the last token (payload start)."""
    toks: list[bytes] = []
    i, n = 2, len(buf)
    while len(toks) < count:
        while i < n and buf[i] in _WS:
            i += 1
        if i < n and buf[i] == ord("#"):
            j = buf.find(b"\n", i)
            i = n if j < 0 else j
            continue
        j = i
        while j < n and buf[j] not in _WS:
            j += 1
        if j == i:
            raise MalformedHeaderError("header ended before all fields were read")
        toks.append(buf[i:j])
        i = j
    if i >= n or buf[i] not in _WS:
        raise MalformedHeaderError("missing whitespace after header")
    return toks, i + 1


def _ints(toks):
    try:
        return [int(t) for t in toks]
    except ValueError as exc:
        raise MalformedHeaderError(f"non-integer header token in {toks}") from exc


def _pgm(buf: bytes) -> np.ndarray:
    toks, start = _header_tokens(buf, 3)
    w, h, maxval = _ints(toks)
    if w < 1 or h < 1:
        raise MalformedHeaderError(f"bad dimensions {w}x{h}")
    if not 0 < maxval <= 65535:
        raise MalformedHeaderError(f"maxval {maxval} outside (0, 65535]")
    if buf[:2] == b"P2":
        words = buf[start - 1:].split()
        if not all(re.fullmatch(rb"[+-]?\d+", t) for t in words):
            raise TruncatedPayloadError("non-integer ASCII sample")
        if len(words) != w * h:
            raise TruncatedPayloadError(f"expected {w * h} samples, found {len(words)}")
        vals = np.array([int(t) for t in words], dtype=np.int64).astype(np.float64)
    else:
        dt = np.dtype(">u2") if maxval > 255 else np.dtype(np.uint8)
        nbytes = w * h * dt.itemsize
        body = buf[start:start + nbytes]
        if len(body) < nbytes:
            raise TruncatedPayloadError(f"expected {nbytes} payload bytes, found {len(body)}")
        vals = np.frombuffer(body, dtype=dt).astype(np.float64)
    if vals.min() < 0 or vals.max() > maxval:
        raise MalformedHeaderError("sample value outside [0, maxval]")
    return (vals / maxval).reshape(h, w)


def _pfm(buf: bytes) -> np.ndarray:
    toks, start = _header_tokens(buf, 3)
    try:
        w, h, scale = int(toks[0]), int(toks[1]), float(toks[2])
    except ValueError as exc:
        raise MalformedHeaderError(f"bad PFM header fields {toks}") from exc
    if w < 1 or h < 1 or scale == 0:
        raise MalformedHeaderError(f"bad PFM header {w}x{h} scale {scale}")
    nbytes = 4 * w * h
    body = buf[start:start + nbytes]
    if len(body) < nbytes:
        raise TruncatedPayloadError(f"expected {nbytes} payload bytes, found {len(body)}")
    vals = np.frombuffer(body, dtype="<f4" if scale < 0 else ">f4").astype(np.float64)
    return np.ascontiguousarray(vals.reshape(h, w)[::-1])  # bottom-to-top scanlines


def read_image(path) -> np.ndarray:
    """PGM (P2/P5) or grayscale PFM file -> float64 image."""
    with open(path, "rb") as fh:
        buf = fh.read()
    magic = buf[:2]
    if magic in (b"P2", b"P5"):
        return _pgm(buf)
    if magic == b"Pf":
        return _pfm(buf)
    raise UnsupportedFormatError(
        f"unsupported magic {magic.decode('ascii', errors='replace')!r} in {path}")


def write_image(img, path, format: str = "pgm8") -> None:  # noqa: A002 (reference name)
    """8-bit binary PGM ('pgm8': clamp, round half up) or float32 PFM ('pfm')."""
    img, _ = A.validate(img, "image")
    img = img.detach().cpu().numpy() if hasattr(img, "detach") else np.asarray(img)
    img = np.asarray(img, dtype=np.float64)
    h, w = img.shape
    fmt = format.lower()
    if fmt == "pgm8":
        q = np.floor(np.clip(img, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
        data = b"P5\n%d %d\n255\n" % (w, h) + q.tobytes()
    elif fmt == "pfm":
        data = b"Pf\n%d %d\n-1.0\n" % (w, h) + np.ascontiguousarray(img[::-1]).astype("<f4").tobytes()
    else:
        raise ValueError(f"unknown format {format!r} (expected 'pgm8' or 'pfm')")
    with open(path, "wb") as fh:
        fh.write(data)
