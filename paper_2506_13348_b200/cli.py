"""Command-line interface on the B200 path (cli.py of the reference; SURVEY.md
§8(f) rank 1).

Subcommands with the reference's names, arguments and JSON summaries:
  render       views of a checkpoint -> PNGs (final, or the 7 decomposition
               buffers with --decompose, computed on the GPU by K14)
  bench-atlas  flat / per-primitive (fp32 software bilinear) / atlas (texture
               units) frame rates, interleaved rounds, CUDA-event timing
               (atlas.py:331-373 bench_matrix; the paper's Table 3)
  pack-atlas   pack a checkpoint's charts and write the atlas pages + sidecar
Every command prints one JSON summary on stdout; errors exit with code 2.

    python -m paper_2506_13348_b200.cli render --scene ckpt --atlas --decompose
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np


def _emit(summary: dict):
    print(json.dumps(summary, indent=2, sort_keys=True))


def _cameras(args):
    from . import formats, synth
    if args.manifest:
        cams, _ = formats.load_manifest(args.manifest)
        return cams
    return synth.camera_ring(1, width=128, height=128)


def write_png(path, img_u8: np.ndarray):
    """8-bit PNG (imgio.py:13-21 after quantisation): (H, W) or (H, W, 3)."""
    from PIL import Image
    Image.fromarray(np.ascontiguousarray(img_u8)).save(path)


DECOMPOSE = (("albedo", 3), ("normal", 3), ("roughness", 1), ("metallic", 1), ("diffuse", 3),
             ("specular", 3), ("final", 3))


def decompose(gbuf_planar, color, diffuse, specular) -> dict:
    """K14: name -> uint8 image (cli.py:70-87 buffers, quantised)."""
    import torch

    from . import _lib
    H, W = int(gbuf_planar.shape[1]), int(gbuf_planar.shape[2])
    out = torch.empty(17 * H * W, dtype=torch.uint8, device=gbuf_planar.device)
    _lib.check(_lib.lib().tsb_decompose(_lib.ptr(gbuf_planar), _lib.ptr(color),
                                        _lib.ptr(diffuse), _lib.ptr(specular), W, H,
                                        _lib.ptr(out), _lib.stream_handle()), "tsb_decompose")
    host = out.cpu().numpy()
    res, o = {}, 0
    for name, ch in DECOMPOSE:
        n = H * W * ch
        res[name] = host[o:o + n].reshape((H, W, 3) if ch == 3 else (H, W))
        o += n
    return res


def cmd_render(args) -> int:
    from . import formats
    from .atlas import pack_atlases
    from .environment import BrdfLut
    from .render import Renderer
    scene = formats.load_scene(args.scene)
    cams = _cameras(args)
    out_dir = Path(args.out or "render_out")
    out_dir.mkdir(parents=True, exist_ok=True)
    lut = BrdfLut.build(device="cuda")
    if args.atlas:
        r = Renderer(scene, pack_atlases(scene), scene.environment, lut, texture_mode="atlas")
    else:
        r = Renderer(scene, None, scene.environment, lut, texture_mode="perprim")
    written = []
    for vi, cam in enumerate(cams):
        color, gbuf = r.render(cam, want_split=True)
        W, H = int(cam.width), int(cam.height)
        _, _, _, dif, spe = r._buffers(W, H)
        imgs = decompose(gbuf.planar, color, dif, spe)
        if args.decompose:
            for name, _ in DECOMPOSE:
                path = out_dir / f"view_{vi:03d}_{name}.png"
                write_png(path, imgs[name])
                written.append(str(path))
        else:
            path = out_dir / f"view_{vi:03d}.png"
            write_png(path, imgs["final"])
            written.append(str(path))
    _emit({"command": "render", "views": len(cams), "atlas": bool(args.atlas),
           "decompose": bool(args.decompose), "files": written})
    return 0


def bench_matrix(scene, cameras, modes=("flat", "perprim", "atlas"), rounds: int = 4) -> dict:
    """atlas.py:331-373 on the GPU: modes timed round-robin, one frame each
    per round (CUDA events around forward + shade), one warmup round; per-mode
    medians and fps ratios."""
    import torch

    from .atlas import pack_atlases
    from .environment import BrdfLut
    from .render import Renderer
    lut = BrdfLut.build(device="cuda")
    atlas_set = pack_atlases(scene) if "atlas" in modes else None
    rend = {m: Renderer(scene, atlas_set if m == "atlas" else None, scene.environment, lut,
                        texture_mode=m) for m in modes}
    times = {m: [] for m in modes}
    frags = {m: 0 for m in modes}
    for rd in range(rounds + 1):
        cam = cameras[rd % len(cameras)]
        for m in modes:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, gb = rend[m].render(cam)
            e1.record()
            torch.cuda.synchronize()
            if rd > 0:
                times[m].append(e0.elapsed_time(e1))
                frags[m] += gb.fragment_count
    out = {}
    for m in modes:
        ms = float(np.median(times[m]))
        out[m] = {"ms_median": ms, "fps": 1e3 / ms if ms > 0 else float("inf"),
                  "fragments_per_frame": frags[m] / rounds}
    out["ratios"] = {f"{a}_vs_{b}": out[a]["fps"] / out[b]["fps"]
                     for a in modes for b in modes if a != b}
    return out


def cmd_bench_atlas(args) -> int:
    from . import synth
    res = args.texture_res if args.texture_res is not None else 16
    seed = args.seed if args.seed is not None else 3
    opts = {"splats": 10000, "views": 2, "width": 128, "rounds": 3}
    if args.config:
        raw = json.loads(Path(args.config).read_text())
        unknown = set(raw) - set(opts)
        if unknown:
            raise SystemExit(f"unknown bench config keys: {sorted(unknown)}")
        opts.update({k: int(v) for k, v in raw.items()})
    print(f"building benchmark scene ({opts['splats']} splats, T={res})...", file=sys.stderr)
    scene = synth.make_shell_scene(opts["splats"], res, seed=seed, with_environment=True)
    cams = synth.bench_cameras(opts["views"], opts["width"], opts["width"])
    m = bench_matrix(scene, cams, rounds=opts["rounds"])
    _emit({"command": "bench-atlas", "texture_res": res, "splats": scene.num_splats,
           "baseline": m["flat"], "software": m["perprim"], "atlas": m["atlas"],
           "atlas_vs_software": m["ratios"]["atlas_vs_perprim"],
           "software_vs_baseline": m["ratios"]["perprim_vs_flat"],
           "atlas_vs_baseline": m["ratios"]["atlas_vs_flat"]})
    return 0


def cmd_pack_atlas(args) -> int:
    from . import formats
    from .atlas import pack_atlases
    scene = formats.load_scene(args.scene)
    a = pack_atlases(scene)
    sidecar = formats.save_atlases(a, Path(args.out or "atlas_out"))
    _emit({"command": "pack-atlas", "splats": scene.num_splats, "resolution": a.resolution,
           "pages": len(a.family_a) + len(a.family_b), "charts_x": a.family_a[0].charts_x,
           "charts_y": a.family_a[0].charts_y, "sidecar": str(sidecar)})
    return 0


def read_png(path) -> np.ndarray:
    """PNG as float64 in [0, 1], (H, W) or (H, W, 3) (imgio.py:24-33)."""
    from PIL import Image
    with Image.open(path) as im:
        if im.mode not in ("L", "RGB"):
            im = im.convert("RGB")
        return np.asarray(im, dtype=np.float64) / 255.0


def _default_init_scene(seed: int):
    """Neutral-material patch when fit gets no initial scene (cli.py:99-108)."""
    from . import synth
    scene = synth.make_plane_scene(nx=6, ny=6, texture_res=1, seed=seed, sh_degree=1,
                                   textured=False, env_levels=4)
    scene.texels[...] = np.array([0.5, 0.5, 0.5, 0.5, 0.05, 0.5, 0.5], np.float32)
    return scene


def _train_config(args):
    """TrainConfig + JSON overrides + --texture-res / --seed (cli.py:111-124)."""
    from .training import TrainConfig
    config = TrainConfig()
    if args.config:
        for key, value in json.loads(Path(args.config).read_text()).items():
            if not hasattr(config, key):
                raise SystemExit(f"unknown config key: {key}")
            setattr(config, key, value)
    if args.texture_res is not None:
        config.texture_resolution = args.texture_res
    if args.seed is not None:
        config.seed = args.seed
    return config


def cmd_fit(args) -> int:
    """Fit a scene to a manifest's images on the GPU (cli.py:127-156): the
    two-stage train() loop, checkpoint, CSV log, final PSNR / SSIM."""
    from . import formats
    from .environment import BrdfLut
    from .training import evaluate, train
    if not args.manifest:
        raise SystemExit("fit requires --manifest")
    cameras, image_paths = formats.load_manifest(args.manifest)
    targets = [read_png(p) for p in image_paths]
    config = _train_config(args)
    init = formats.load_scene(args.scene) if args.scene else _default_init_scene(config.seed)
    out_dir = Path(args.out or "fit_out")
    out_dir.mkdir(parents=True, exist_ok=True)
    lut = BrdfLut.build(device="cuda")
    fitted, history = train(init, cameras, targets, config, lut,
                            log_path=out_dir / "train_log.csv")
    formats.save_scene(fitted, out_dir / "scene")
    final = evaluate(fitted, cameras, targets, lut)
    _emit({"command": "fit", "iterations": config.iterations, "splats": fitted.num_splats,
           "loss": history[-1]["loss"] if history else None, "psnr": final["psnr"],
           "ssim": final["ssim"], "checkpoint": str(out_dir / "scene"),
           "log": str(out_dir / "train_log.csv")})
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="texsplat-b200",
                                     description="Textured 2D Gaussian splats on B200.")
    sub = parser.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--scene", help="scene directory")
        p.add_argument("--manifest", help="dataset manifest JSON")
        p.add_argument("--out", help="output directory")
        p.add_argument("--atlas", action="store_true", help="sample textures through atlases")
        p.add_argument("--decompose", action="store_true", help="also write per-buffer images")
        p.add_argument("--texture-res", type=int, default=None)
        p.add_argument("--seed", type=int, default=None)
        p.add_argument("--threads", type=int, default=None, help="accepted; the GPU is the pool")
        p.add_argument("--config", help="JSON config overrides")

    for name, fn in (("render", cmd_render), ("fit", cmd_fit), ("bench-atlas", cmd_bench_atlas),
                     ("pack-atlas", cmd_pack_atlas)):
        p = sub.add_parser(name)
        common(p)
        p.set_defaults(fn=fn)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (OSError, ValueError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
