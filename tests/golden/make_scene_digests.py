"""Writes tests/golden/scene_digests.json: SHA-256 of every BASELINE config's
seeded synthetic object and mask bytes (paper_2211_09938_b200/scenes.py) and
the realised nonzero / salient fractions.

  python tests/golden/make_scene_digests.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2211_09938_b200 import scenes  # noqa: E402


def main() -> None:
    out = {}
    for name, cfg, frac in scenes.digest_cases():
        out[name] = scenes.scene_digest(scenes.make_scene(cfg, saliency_frac=frac))
    path = Path(__file__).with_name("scene_digests.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(path)


if __name__ == "__main__":
    main()
