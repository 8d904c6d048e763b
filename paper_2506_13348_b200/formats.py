"""On-disk formats of the reference, read straight into device memory
(SURVEY.md §8(f) rank 3).

Byte-compatible readers and writers for:
  * scene checkpoints: scene.json master + TSPL splat blob (float64 SoA) +
    TTEX texel blob (float32, combined order) + PFM environment
    (scene.py:154-285, textures.py:371-408, imgio.py:33-66)
  * atlas pages: PFM rgb/a page files + JSON sidecar (atlas.py:214-281)
  * dataset manifests (scene.py:288-343)
The blobs are parsed with np.frombuffer views (no per-splat Python objects —
the reference builds one MaterialTextureSet per splat) and uploaded with one
copy per array; `load_scene_device` returns the DeviceScene and the (P,T,T,7)
texel tensor ready for the render path. Errors follow the reference:
SchemaError / VersionError (ValueError), MissingReferenceError
(FileNotFoundError).
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .atlas import FAMILY_A, FAMILY_B, AtlasSet, IndirectionBuffer, TextureAtlas
from .environment import EnvironmentLight
from .scene import Scene, TextureConfig
from .splats import Camera

SCENE_VERSION = 1
MANIFEST_VERSION = 1
SPLATS_MAGIC = b"TSPL"
BLOB_MAGIC = b"TTEX"
COMBINED_CHANNELS = 7


class SchemaError(ValueError):
    pass


class VersionError(ValueError):
    pass


class MissingReferenceError(FileNotFoundError):
    pass


# ---------------------------------------------------------------------------
# PFM (imgio.py:33-66)
# ---------------------------------------------------------------------------
def write_pfm(path, data):
    """float32 PFM, 'Pf' for (H, W), 'PF' for (H, W, 3), bottom-to-top rows,
    little endian (negative scale)."""
    data = np.asarray(data, dtype=np.float32)
    if data.ndim == 2:
        header = b"Pf"
    elif data.ndim == 3 and data.shape[2] == 3:
        header = b"PF"
    else:
        raise ValueError("PFM holds 1- or 3-channel images")
    with open(path, "wb") as f:
        f.write(header + b"\n")
        f.write(f"{data.shape[1]} {data.shape[0]}\n".encode())
        f.write(b"-1.0\n")
        f.write(np.ascontiguousarray(data[::-1], dtype="<f4").tobytes())


def read_pfm(path) -> np.ndarray:
    with open(path, "rb") as f:
        kind = f.readline().strip()
        if kind == b"PF":
            channels = 3
        elif kind == b"Pf":
            channels = 1
        else:
            raise ValueError(f"not a PFM file: header {kind!r}")
        dims = f.readline().split()
        w, h = int(dims[0]), int(dims[1])
        scale = float(f.readline().strip())
        count = w * h * channels
        raw = np.frombuffer(f.read(count * 4), dtype="<f4" if scale < 0 else ">f4", count=count)
    shape = (h, w) if channels == 1 else (h, w, channels)
    return raw.reshape(shape)[::-1].astype(np.float32)


# ---------------------------------------------------------------------------
# TSPL / TTEX blobs
# ---------------------------------------------------------------------------
def write_splats_blob(path, positions, tangent_u, tangent_v, scales, opacities, sh):
    """scene.py:154-161: 'TSPL', <u32 version, count, K>, then the six
    float64 arrays back to back."""
    count, k = int(np.asarray(positions).shape[0]), int(np.asarray(sh).shape[1])
    with open(path, "wb") as f:
        f.write(SPLATS_MAGIC)
        f.write(struct.pack("<III", SCENE_VERSION, count, k))
        for arr in (positions, tangent_u, tangent_v, scales, opacities, sh):
            f.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def read_splats_blob(path):
    """Returns (positions, tangent_u, tangent_v, scales, opacities, sh) as
    float64 views of one buffer (scene.py:164-186)."""
    raw = Path(path).read_bytes()
    if raw[:4] != SPLATS_MAGIC:
        raise SchemaError(f"bad splat blob magic {raw[:4]!r}")
    version, count, k = struct.unpack("<III", raw[4:16])
    if version != SCENE_VERSION:
        raise VersionError(f"splat blob version {version} unsupported")
    sizes = [count * 3, count * 3, count * 3, count * 2, count, count * k * 3]
    if len(raw) - 16 != sum(sizes) * 8:
        raise SchemaError("splat blob payload size mismatch")
    flat = np.frombuffer(raw, dtype="<f8", offset=16)
    out, off = [], 0
    for n in sizes:
        out.append(flat[off:off + n])
        off += n
    pos, tu, tv, sc, op, sh = out
    return (pos.reshape(count, 3), tu.reshape(count, 3), tv.reshape(count, 3),
            sc.reshape(count, 2), op, sh.reshape(count, k, 3))


def write_texture_blob(path, texels):
    """textures.py:371-392: 'TTEX', <u32 T, 7, count>, then count blocks of
    (T, T, 7) float32 in combined order."""
    texels = np.asarray(texels, dtype=np.float32)
    if texels.ndim != 4 or texels.shape[3] != COMBINED_CHANNELS or texels.shape[0] == 0:
        raise ValueError("no texture sets to save")
    with open(path, "wb") as f:
        f.write(BLOB_MAGIC)
        f.write(struct.pack("<III", texels.shape[1], COMBINED_CHANNELS, texels.shape[0]))
        f.write(np.ascontiguousarray(texels, dtype="<f4").tobytes())


def read_texture_blob(path) -> np.ndarray:
    """(count, T, T, 7) float32 view (textures.py:395-408)."""
    raw = Path(path).read_bytes()
    if raw[:4] != BLOB_MAGIC:
        raise ValueError(f"bad texture blob magic {raw[:4]!r}")
    T, Cc, count = struct.unpack("<III", raw[4:16])
    if Cc != COMBINED_CHANNELS:
        raise ValueError(f"texture blob has {Cc} channels, expected 7")
    if len(raw) - 16 != count * T * T * Cc * 4:
        raise ValueError("texture blob payload size mismatch")
    return np.frombuffer(raw, dtype="<f4", offset=16).reshape(count, T, T, Cc)


# ---------------------------------------------------------------------------
# scene checkpoints (scene.py:189-285)
# ---------------------------------------------------------------------------
def save_scene(scene: Scene, out_dir) -> Path:
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    write_splats_blob(out_dir / "scene.splats.bin", scene.positions, scene.tangent_u,
                      scene.tangent_v, scene.scales, scene.opacities, scene.sh)
    write_texture_blob(out_dir / "scene.textures.bin", scene.texels)
    meta = {
        "version": SCENE_VERSION,
        "num_splats": scene.num_splats,
        "sh_degree": scene.sh_degree,
        "texture_resolution": scene.texture_config.resolution,
        "texture_support": scene.texture_config.support,
        "background": [float(x) for x in scene.background],
        "splats": "scene.splats.bin",
        "textures": "scene.textures.bin",
    }
    if scene.environment is not None:
        env = scene.environment
        meta["environment"] = {"levels": env.levels,
                               "spec": [f"env.spec{i}.pfm" for i in range(env.levels)],
                               "diffuse": "env.diffuse.pfm"}
        for i, mip in enumerate(env.spec_mips):
            write_pfm(out_dir / f"env.spec{i}.pfm", mip)
        write_pfm(out_dir / "env.diffuse.pfm", env.diffuse)
    if scene.mesh is not None:
        raise NotImplementedError("mesh visibility is outside the B200 render path")
    path = out_dir / "scene.json"
    with open(path, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    return path


def _require(directory: Path, name: str) -> Path:
    p = directory / name
    if not p.exists():
        raise MissingReferenceError(f"scene references missing file {name}")
    return p


def _read_master(path):
    path = Path(path)
    if path.is_dir():
        path = path / "scene.json"
    if not path.exists():
        raise MissingReferenceError(f"no scene file at {path}")
    try:
        meta = json.loads(path.read_text())
    except json.JSONDecodeError as e:
        raise SchemaError(f"scene master is not valid JSON: {e}") from e
    if meta.get("version") != SCENE_VERSION:
        raise VersionError(f"scene version {meta.get('version')} unsupported")
    return meta, path.parent


def load_scene(path) -> Scene:
    """Read a reference checkpoint (scene.py:234-285) into a host Scene."""
    meta, directory = _read_master(path)
    pos, tu, tv, sc, op, sh = read_splats_blob(_require(directory, meta["splats"]))
    texels = read_texture_blob(_require(directory, meta["textures"]))
    if texels.shape[0] != pos.shape[0]:
        raise SchemaError("texture count does not match splat count")
    t_res = int(meta["texture_resolution"])
    if texels.shape[0] and texels.shape[1] != t_res:
        raise SchemaError("texture blob resolution mismatch with master")
    env = None
    if "environment" in meta:
        e = meta["environment"]
        env = EnvironmentLight([read_pfm(_require(directory, n)) for n in e["spec"]],
                               read_pfm(_require(directory, e["diffuse"])))
    if "mesh" in meta:
        raise NotImplementedError("mesh visibility is outside the B200 render path")
    pos, tu, tv, sc, op, sh, texels = (np.array(a) for a in (pos, tu, tv, sc, op, sh, texels))
    return Scene(pos, tu, tv, sc, op, sh, int(meta["sh_degree"]), texels,
                 TextureConfig(t_res, float(meta["texture_support"])), env, None,
                 np.asarray(meta["background"], dtype=np.float64))


def load_scene_device(path, device="cuda"):
    """Checkpoint straight to HBM: (DeviceScene, texels (P,T,T,7) float32
    device tensor, EnvironmentLight or None, background, meta). One upload per
    array from the blob views; no host Scene or per-splat objects."""
    import torch

    from .device import DeviceScene
    meta, directory = _read_master(path)
    arrs = read_splats_blob(_require(directory, meta["splats"]))
    texels = read_texture_blob(_require(directory, meta["textures"]))
    if texels.shape[0] != arrs[0].shape[0]:
        raise SchemaError("texture count does not match splat count")
    t_res = int(meta["texture_resolution"])
    dev = torch.device(device)
    up = [torch.from_numpy(np.array(a, dtype=np.float64)).to(dev) for a in arrs]
    ds = DeviceScene.from_tensors(*up, int(meta["sh_degree"]), t_res)
    tex = torch.from_numpy(np.array(texels, dtype=np.float32)).to(dev)
    env = None
    if "environment" in meta:
        e = meta["environment"]
        env = EnvironmentLight([read_pfm(_require(directory, n)) for n in e["spec"]],
                               read_pfm(_require(directory, e["diffuse"])))
    return ds, tex, env, np.asarray(meta["background"], dtype=np.float64), meta


def prepare_device(dscene, texels):
    """PreparedScene (fp32 software-bilinear sampler) over device-resident
    texels (P, T, T, 7): the charts are interleaved into the 8-channel atlas
    order on the device — no host packing."""
    import torch

    from .device import DeviceAtlas, FrameWorkspace
    from .rasterize import PreparedScene
    P, T = int(texels.shape[0]), int(texels.shape[1])
    t8 = torch.zeros((P, T, T, 8), dtype=torch.float32, device=texels.device)
    t8[..., [0, 1, 2, 3, 6, 4, 5]] = texels
    return PreparedScene(dscene, DeviceAtlas.interleaved(t8), "perprim", "verify",
                         workspace=FrameWorkspace(texels.device))


# ---------------------------------------------------------------------------
# atlas pages (atlas.py:214-281)
# ---------------------------------------------------------------------------
def save_atlases(atlas_set: AtlasSet, out_dir, stem: str = "atlas") -> Path:
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    pages = []
    for page in atlas_set.atlases:
        base = f"{stem}.{page.family}.{page.page_index}"
        write_pfm(out_dir / f"{base}.rgb.pfm", page.texels[:, :, 0:3])
        write_pfm(out_dir / f"{base}.a.pfm", page.texels[:, :, 3])
        pages.append({"family": page.family, "page": page.page_index,
                      "rgb": f"{base}.rgb.pfm", "a": f"{base}.a.pfm"})
    ind = atlas_set.indirection
    sidecar = {
        "resolution": atlas_set.resolution,
        "charts_x": ind.charts_x,
        "charts_y": ind.charts_y,
        "pages": len(atlas_set.family_a),
        "page_files": pages,
        "indirection": {str(i): [int(p), int(cx), int(cy)]
                        for i, (cx, cy, p) in enumerate(ind.entries)},
    }
    side_path = out_dir / f"{stem}.json"
    with open(side_path, "w") as f:
        json.dump(sidecar, f, indent=1, sort_keys=True)
    return side_path


def load_atlases(sidecar_path) -> AtlasSet:
    sidecar_path = Path(sidecar_path)
    with open(sidecar_path) as f:
        meta = json.load(f)
    directory = sidecar_path.parent
    T = int(meta["resolution"])
    charts_x, charts_y, n_pages = int(meta["charts_x"]), int(meta["charts_y"]), int(meta["pages"])
    fam = {FAMILY_A: [None] * n_pages, FAMILY_B: [None] * n_pages}
    for entry in meta["page_files"]:
        rgb = read_pfm(directory / entry["rgb"])
        a = read_pfm(directory / entry["a"])
        texels = np.concatenate([rgb, a[:, :, None]], axis=2).astype(np.float32)
        page = TextureAtlas(texels, entry["family"], int(entry["page"]), charts_x, charts_y, T)
        fam[entry["family"]][page.page_index] = page
    ids = sorted(meta["indirection"], key=int)
    entries = np.zeros((len(ids), 3), dtype=np.int32)
    for sid in ids:
        p, cx, cy = meta["indirection"][sid]
        entries[int(sid)] = (cx, cy, p)
    return AtlasSet(fam[FAMILY_A], fam[FAMILY_B],
                    IndirectionBuffer(entries, charts_x, charts_y, n_pages), T)


# ---------------------------------------------------------------------------
# manifests (scene.py:288-343)
# ---------------------------------------------------------------------------
def save_manifest(path, cameras, image_names):
    if len(cameras) != len(image_names):
        raise ValueError("need one image per camera")
    if not cameras:
        raise ValueError("empty dataset")
    c0 = cameras[0]
    for c in cameras:
        if (c.fx, c.fy, c.cx, c.cy, c.width, c.height) != \
                (c0.fx, c0.fy, c0.cx, c0.cy, c0.width, c0.height):
            raise ValueError("manifest cameras must share intrinsics")
    meta = {"version": MANIFEST_VERSION,
            "intrinsics": {"fx": c0.fx, "fy": c0.fy, "cx": c0.cx, "cy": c0.cy,
                           "width": c0.width, "height": c0.height,
                           "near": c0.near, "far": c0.far},
            "views": [{"image": name, "world_to_view": cam.world_to_view.tolist()}
                      for cam, name in zip(cameras, image_names)]}
    with open(path, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def load_manifest(path):
    path = Path(path)
    if not path.exists():
        raise MissingReferenceError(f"no manifest at {path}")
    try:
        meta = json.loads(path.read_text())
    except json.JSONDecodeError as e:
        raise SchemaError(f"manifest is not valid JSON: {e}") from e
    if meta.get("version") != MANIFEST_VERSION:
        raise VersionError(f"manifest version {meta.get('version')} unsupported")
    try:
        intr, views = meta["intrinsics"], meta["views"]
    except KeyError as e:
        raise SchemaError(f"manifest missing key {e}") from e
    cams, images = [], []
    for v in views:
        cams.append(Camera(np.asarray(v["world_to_view"], dtype=np.float64),
                           fx=float(intr["fx"]), fy=float(intr["fy"]), cx=float(intr["cx"]),
                           cy=float(intr["cy"]), width=int(intr["width"]),
                           height=int(intr["height"]), near=float(intr.get("near", 0.01)),
                           far=float(intr.get("far", 100.0))))
        images.append(path.parent / v["image"])
    return cams, images
