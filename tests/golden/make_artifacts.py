"""Generate the committed `.lut` container fixtures from the REFERENCE itself.

Run in the build container, where /root/reference exists:
    make -C oracle ref && python tests/golden/make_artifacts.py
It loads oracle/_ref/liblutkan_ref.so (the reference's own sources, artifact_io.cpp and
detail/zip.cpp included) and writes, under tests/golden/artifacts/:
  * reference-written archives (save_artifact, artifact_io.cpp:206-219) of small recipe layers,
  * corrupted / malformed variants of one of them, each with the status the reference's
    load_artifact returns for it (artifact_io.cpp:221-300; codes as in include/lutkan_b200.h),
recorded in artifacts.json. tests/test_artifact_io.py pins lkg_artifact_save / _load / _check to
these when the reference library is absent (the GPU box).
"""
from __future__ import annotations

import io
import json
import os
import struct
import sys
import zipfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "artifacts")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.pyoracle import Oracle  # noqa: E402

# (file, cfg, layer, L, scheme, value_repr, param_dtype, boundary_mode, oob_policy)
ARCHIVES = [("c1_sym_sr.lut", 1, 0, 16, 0, 1, 0, 1, 0), ("c1_asym_phi_f16.lut", 1, 0, 16, 1, 0, 1, 0, 1),
            ("c1_asym_sr_f16_zs.lut", 1, 1, 32, 1, 1, 1, 1, 1), ("c2_sym_sr_l1.lut", 2, 1, 64, 0, 1, 0, 1, 0)]


def entries(raw: bytes) -> dict:
    z = zipfile.ZipFile(io.BytesIO(raw))
    return {i.filename: z.read(i.filename) for i in z.infolist()}


def rezip(ents: dict, order=None) -> bytes:
    b = io.BytesIO()
    with zipfile.ZipFile(b, "w", compression=zipfile.ZIP_DEFLATED) as z:
        for k in order or ents:
            z.writestr(k, ents[k])
    return b.getvalue()


def with_manifest(raw: bytes, edit) -> bytes:
    ents = entries(raw)
    m = json.loads(ents["manifest.json"])
    edit(m)
    ents["manifest.json"] = json.dumps(m, indent=2, sort_keys=True).encode()
    return rezip(ents)


def central_offset(raw: bytes, name: str) -> int:
    end = raw.rfind(b"PK\x05\x06")
    cd = struct.unpack_from("<I", raw, end + 16)[0]
    off = cd
    while raw[off:off + 4] == b"PK\x01\x02":
        nl, xl, cl = struct.unpack_from("<HHH", raw, off + 28)
        if raw[off + 46:off + 46 + nl].decode() == name:
            return off
        off += 46 + nl + xl + cl
    raise KeyError(name)


def local_offset(raw: bytes, name: str) -> int:
    return struct.unpack_from("<I", raw, central_offset(raw, name) + 42)[0]


def corruptions(base: bytes) -> dict:
    c = {}
    c["truncated"] = base[: len(base) // 2]
    c["tiny"] = base[:10]
    b = bytearray(base)
    b[central_offset(base, "knots.bin")] ^= 0xFF
    c["bad_central_sig"] = bytes(b)
    b = bytearray(base)
    b[local_offset(base, "scale.bin")] ^= 0xFF
    c["bad_local_sig"] = bytes(b)
    b = bytearray(base)
    lo = local_offset(base, "q_table.bin")
    nl, xl = struct.unpack_from("<HH", base, lo + 26)
    b[lo + 30 + nl + xl + 40] ^= 0x5A
    c["payload_flip"] = bytes(b)
    b = bytearray(base)
    co = central_offset(base, "knots.bin")
    struct.pack_into("<I", b, co + 16, struct.unpack_from("<I", base, co + 16)[0] ^ 1)
    c["crc_mismatch"] = bytes(b)
    b = bytearray(base)
    struct.pack_into("<H", b, central_offset(base, "scale.bin") + 10, 12)
    c["bad_method"] = bytes(b)
    c["version"] = with_manifest(base, lambda m: m.update(format_version="lutkan/2"))
    c["enum_scheme"] = with_manifest(base, lambda m: m.update(scheme="foo"))
    c["enum_boundary"] = with_manifest(base, lambda m: m.update(boundary_mode="open"))
    c["missing_L"] = with_manifest(base, lambda m: m.pop("L"))
    c["missing_blob_decl"] = with_manifest(base, lambda m: m["blobs"].pop("y_min"))
    c["int_as_string"] = with_manifest(base, lambda m: m.update(in_dim=str(m["in_dim"])))
    c["real_for_int"] = with_manifest(base, lambda m: m.update(L=float(m["L"])))
    c["shape_mismatch"] = with_manifest(base, lambda m: m["blobs"]["q_table"]["shape"].__setitem__(2, m["L"] + 1))
    c["shape_rank"] = with_manifest(base, lambda m: m["blobs"]["scale"]["shape"].append(1))
    c["dtype_mismatch"] = with_manifest(base, lambda m: m["blobs"]["scale"].update(dtype="f16"))
    c["segments_zero"] = with_manifest(base, lambda m: m.update(segments=0))
    c["blobs_not_object"] = with_manifest(base, lambda m: m.update(blobs=[1, 2]))
    c["base_kind_tanh"] = with_manifest(base, lambda m: m.update(base_kind="tanh"))
    c["base_kind_missing"] = with_manifest(base, lambda m: m.pop("base_kind"))
    ents = entries(base)
    ents["y_min.bin"] = ents["y_min.bin"][:-4]
    c["blob_size"] = rezip(ents)
    ents = entries(base)
    ents.pop("y_min.bin")
    c["missing_entry"] = rezip(ents)
    ents = entries(base)
    c["no_manifest"] = rezip({k: v for k, v in ents.items() if k != "manifest.json"})
    ents = entries(base)
    ents["manifest.json"] = b"{\n  \"L\": 16,"
    c["not_json"] = rezip(ents)
    ents = entries(base)
    ents["manifest.json"] = b"[1, 2]"
    c["not_object"] = rezip(ents)
    ents = entries(base)
    kn = np.frombuffer(ents["knots.bin"], np.float32).copy()
    kn[[1, 2]] = kn[[2, 1]]
    ents["knots.bin"] = kn.tobytes()
    c["knots_unsorted"] = rezip(ents)
    kn[[1, 2]] = kn[[2, 1]]
    kn[3] = np.nan
    ents["knots.bin"] = kn.tobytes()
    c["knots_nan"] = rezip(ents)
    ents = entries(base)
    order = ["edge_out_scale.bin"] + [k for k in ents if k != "edge_out_scale.bin"]
    c["reordered_entries"] = rezip(ents, order)  # entry order is free on read
    return c


def main():
    o = Oracle("reference")
    assert o.kind == "reference"
    os.makedirs(os.path.join(OUT, "corrupt"), exist_ok=True)
    rec = {"generator": "tests/golden/make_artifacts.py", "archives": [], "corrupt": []}
    for name, cfg, layer, L, scheme, vr, pd, bm, op in ARCHIVES:
        art = o.compile_layer(o.recipe_layer(cfg, layer), L, scheme, vr, pd, bm, op)
        path = os.path.join(OUT, name)
        o.artifact_save(art, path)
        assert o.artifact_load_status(path) == 0
        rec["archives"].append(dict(file=name, cfg=cfg, layer=layer, L=L, scheme=scheme, value_repr=vr,
                                    param_dtype=pd, boundary_mode=bm, oob_policy=op))
    base = open(os.path.join(OUT, "c1_sym_sr.lut"), "rb").read()
    for cname, raw in corruptions(base).items():
        path = os.path.join(OUT, "corrupt", cname + ".lut")
        with open(path, "wb") as f:
            f.write(raw)
        rec["corrupt"].append(dict(file="corrupt/" + cname + ".lut", status=int(o.artifact_load_status(path))))
    with open(os.path.join(OUT, "artifacts.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print("\n".join(f"{c['file']}: {c['status']}" for c in rec["corrupt"]))


if __name__ == "__main__":
    main()
