"""``.nolf`` asset files: the on-disk input of the render path.

Format (reference assetio.py:1-7, 30-66): magic ``NOLF``, ``<HH`` version and
section count, then per section ``name[16] <QQI offset, length, crc32``, then
the raw little-endian section bytes; array shapes and scalars live in the
JSON ``meta`` section (assetio.py:85-158).  ``read_asset`` returns this
package's ``LightFieldAsset`` (model.py); gzip-compressed files are accepted.
"""

from __future__ import annotations

import gzip
import json
import struct
import zlib
from pathlib import Path

import numpy as np

from . import errors
from .model import (Aabb, CubeAtlas, HashGridEncoder, LightFieldAsset, MarchParams, Mlp,
                    ModelWiring, PshTable)

MAGIC = b"NOLF"
VERSION = 1
_NAME = 16
_ENTRY = struct.Struct("<QQI")


def unpack_sections(data: bytes) -> dict:
    if data[:4] != MAGIC:
        raise errors.DataError("not an asset file (bad magic)")
    if len(data) < 8:
        raise errors.DataError("asset header truncated")
    version, count = struct.unpack_from("<HH", data, 4)
    if version != VERSION:
        raise errors.DataError(f"unsupported asset version {version}")
    out = {}
    pos = 8
    for _ in range(count):
        if pos + _NAME + _ENTRY.size > len(data):
            raise errors.DataError("section table truncated")
        name = data[pos:pos + _NAME].rstrip(b"\0").decode("ascii")
        off, length, crc = _ENTRY.unpack_from(data, pos + _NAME)
        pos += _NAME + _ENTRY.size
        blob = data[off:off + length]
        if len(blob) != length:
            raise errors.DataError(f"section {name} truncated")
        if zlib.crc32(blob) != crc:
            raise errors.DataError(f"section {name} failed its checksum")
        out[name] = blob
    return out


def pack_sections(sections: dict) -> bytes:
    header = 8 + len(sections) * (_NAME + _ENTRY.size)
    table, blobs, off = [], [], header
    for name, blob in sections.items():
        raw = name.encode("ascii")
        if len(raw) > _NAME:
            raise errors.DataError(f"section name too long: {name}")
        table.append(raw.ljust(_NAME, b"\0") + _ENTRY.pack(off, len(blob), zlib.crc32(blob)))
        blobs.append(blob)
        off += len(blob)
    return MAGIC + struct.pack("<HH", VERSION, len(sections)) + b"".join(table) + b"".join(blobs)


def _arr(sections, name, dtype, shape):
    if name not in sections:
        raise errors.DataError(f"missing section {name}")
    a = np.frombuffer(sections[name], dtype=np.dtype(dtype).newbyteorder("<"))
    if a.size != int(np.prod(shape)):
        raise errors.DataError(f"section {name} has {a.size} elements, expected {shape}")
    return a.reshape(shape).astype(dtype)


def _mlp(meta, sections, tag) -> Mlp:
    widths = meta["widths"]
    ws = [_arr(sections, f"{tag}_w{i}", np.float32, (widths[i + 1], widths[i]))
          for i in range(len(widths) - 1)]
    bs = [_arr(sections, f"{tag}_b{i}", np.float32, (widths[i + 1],))
          for i in range(len(widths) - 1)]
    return Mlp(weights=ws, biases=bs, heads=tuple((a, int(w)) for a, w in meta["heads"]))


def read_asset(path_or_bytes) -> LightFieldAsset:
    if isinstance(path_or_bytes, (bytes, bytearray, memoryview)):
        data = bytes(path_or_bytes)
    else:
        data = Path(path_or_bytes).read_bytes()
    if data[:2] == b"\x1f\x8b":
        data = gzip.decompress(data)
    s = unpack_sections(data)
    try:
        meta = json.loads(s["meta"].decode("utf-8"))
    except (KeyError, json.JSONDecodeError) as e:
        raise errors.DataError(f"bad asset meta section: {e}") from e
    pm = meta["psh"]
    psh = PshTable(resolution=pm["resolution"], table_size=pm["table_size"],
                   offset_size=pm["offset_size"],
                   offsets=_arr(s, "psh_offsets", np.int64, (pm["offset_size"],)),
                   report=pm.get("report"),
                   primes_h0=np.array(pm["primes_h0"], dtype=np.uint64),
                   primes_h1=np.array(pm["primes_h1"], dtype=np.uint64))
    feats = _arr(s, "psh_features", np.float32, (pm["table_size"], pm["features"]))

    def atlas(m, tag, ch):
        return CubeAtlas(base_resolution=m["b"], cube_resolution=m["r"], channels=ch,
                         index=_arr(s, f"{tag}_index", np.int32, (m["b"],) * 3),
                         cubes=_arr(s, f"{tag}_cubes", np.float32,
                                    (m["cubes"], m["r"] + 1, m["r"] + 1, m["r"] + 1, ch)))

    den = atlas(meta["density_atlas"], "den", 1)
    dif = atlas(meta["diffuse_atlas"], "dif", 4) if meta.get("has_diffuse_atlas") else None
    em = meta["diffuse_encoder"]
    enc = HashGridEncoder(levels=em["levels"], base_resolution=em["base_resolution"],
                          growth=em["growth"], table_size=em["table_size"],
                          features_per_level=em["features_per_level"])
    dfeat = [_arr(s, f"ed_feat_{i}", np.float32, (rows, em["features_per_level"]))
             for i, rows in enumerate(enc.row_counts)]
    mm, wm = meta["march"], meta["wiring"]
    mesh = None
    if "proxy_mesh" in meta:      # extension section (not written by the reference)
        pm2 = meta["proxy_mesh"]
        mesh = (_arr(s, "mesh_vertices", np.float64, (pm2["vertices"], 3)),
                _arr(s, "mesh_triangles", np.int32, (pm2["triangles"], 3)))
    return LightFieldAsset(
        density_atlas=den, psh=psh, psh_features=feats, diffuse_encoder=enc,
        diffuse_features=dfeat, specular_mlp=_mlp(meta["specular_mlp"], s, "fs"),
        diffuse_mlp=_mlp(meta["diffuse_mlp"], s, "fd"),
        march=MarchParams(step=mm["step"], t_stop=mm["t_stop"], alpha_floor=mm["alpha_floor"]),
        proxy=Aabb(min=np.array(meta["proxy"]["min"]), max=np.array(meta["proxy"]["max"])),
        object_to_world=np.array(meta["transform"], dtype=np.float64).reshape(4, 4),
        diffuse_atlas=dif, wiring=ModelWiring(**wm), name=meta.get("name", "asset"),
        proxy_mesh=mesh)


def _le(a: np.ndarray) -> bytes:
    return np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<")).tobytes()


def write_asset(asset, path=None) -> bytes:
    """Serialise any attribute-compatible asset; returns the bytes and writes
    them to ``path`` when given (assetio.py:85-158 layout)."""
    if asset.density_atlas is None:
        raise errors.DataError("analytic assets have no serialized form")

    def mlp_meta(m):
        return {"widths": [m.weights[0].shape[1]] + [w.shape[0] for w in m.weights],
                "heads": [[a, w] for a, w in m.heads]}

    rep = asset.psh.report
    if rep is not None and not isinstance(rep, dict):
        rep = {"load_factor": rep.load_factor, "adjacency_score": rep.adjacency_score,
               "attempts": rep.attempts}
    enc = asset.diffuse_encoder
    meta = {
        "name": asset.name,
        "march": {"step": asset.march.step, "t_stop": asset.march.t_stop,
                  "alpha_floor": asset.march.alpha_floor},
        "wiring": {k: bool(getattr(asset.wiring, k)) for k in
                   ("use_hit_point", "use_opacity", "refine_opacity", "use_tint",
                    "use_diffuse_color")},
        "proxy": {"min": np.asarray(asset.proxy.min).tolist(),
                  "max": np.asarray(asset.proxy.max).tolist()},
        "transform": np.asarray(asset.object_to_world, np.float64).reshape(-1).tolist(),
        "density_atlas": {"b": asset.density_atlas.base_resolution,
                          "r": asset.density_atlas.cube_resolution,
                          "cubes": len(asset.density_atlas.cubes)},
        "psh": {"resolution": asset.psh.resolution, "table_size": asset.psh.table_size,
                "offset_size": asset.psh.offset_size,
                "primes_h0": np.asarray(asset.psh.primes_h0, np.uint64).tolist(),
                "primes_h1": np.asarray(asset.psh.primes_h1, np.uint64).tolist(),
                "features": asset.psh_features.shape[1],
                "report": rep or {"load_factor": 0.0, "adjacency_score": 0.0, "attempts": 0}},
        "diffuse_encoder": {"levels": enc.levels, "base_resolution": enc.base_resolution,
                            "growth": enc.growth, "table_size": enc.table_size,
                            "features_per_level": enc.features_per_level},
        "specular_mlp": mlp_meta(asset.specular_mlp),
        "diffuse_mlp": mlp_meta(asset.diffuse_mlp),
        "has_diffuse_atlas": asset.diffuse_atlas is not None,
    }
    mesh = getattr(asset, "proxy_mesh", None)
    if mesh is not None:
        meta["proxy_mesh"] = {"vertices": int(len(mesh[0])), "triangles": int(len(mesh[1]))}
    if asset.diffuse_atlas is not None:
        meta["diffuse_atlas"] = {"b": asset.diffuse_atlas.base_resolution,
                                 "r": asset.diffuse_atlas.cube_resolution,
                                 "cubes": len(asset.diffuse_atlas.cubes)}
    sec = {
        "meta": json.dumps(meta).encode("utf-8"),
        "psh_offsets": _le(np.asarray(asset.psh.offsets, np.int64)),
        "psh_features": _le(np.asarray(asset.psh_features, np.float32)),
        "den_index": _le(np.asarray(asset.density_atlas.index, np.int32)),
        "den_cubes": _le(np.asarray(asset.density_atlas.cubes, np.float32)),
    }
    if asset.diffuse_atlas is not None:
        sec["dif_index"] = _le(np.asarray(asset.diffuse_atlas.index, np.int32))
        sec["dif_cubes"] = _le(np.asarray(asset.diffuse_atlas.cubes, np.float32))
    for i, f in enumerate(asset.diffuse_features):
        sec[f"ed_feat_{i}"] = _le(np.asarray(f, np.float32))
    for tag, m in (("fs", asset.specular_mlp), ("fd", asset.diffuse_mlp)):
        for i, w in enumerate(m.weights):
            sec[f"{tag}_w{i}"] = _le(np.asarray(w, np.float32))
        for i, b in enumerate(m.biases):
            sec[f"{tag}_b{i}"] = _le(np.asarray(b, np.float32))
    if mesh is not None:
        sec["mesh_vertices"] = _le(np.asarray(mesh[0], np.float64).reshape(-1, 3))
        sec["mesh_triangles"] = _le(np.asarray(mesh[1], np.int32).reshape(-1, 3))
    data = pack_sections(sec)
    if path is not None:
        Path(path).write_bytes(data)
    return data
