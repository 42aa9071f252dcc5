"""Golden parse errors: each malformed scene snippet through the reference's own
loadSceneFile (oracle/_ref/ref_parity scene), recording its SceneParseError text
-> tests/golden_parse_errors.json (used by tests/test_scene_file.py)."""
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
EXE = os.path.join(HERE, "_ref", "ref_parity")

SNIPPETS = [
    "primitive { kind cone size 1 }",
    "primitive { kind box size 1 2 }",
    "primitive { kind sphere size -1 }",
    "primitive { kind sphere size 1 id 3 }\nprimitive { kind sphere size 2 id 3 }",
    "primitive { kind sphere size 1 albedo 1.5 0 0 }",
    "camera { fov_y 200 }",
    "camera { zoom 2 }",
    "config { hysteresis 1.5 }",
    "config { n_rays 4 }",
    "config { max_trace_steps 1.5 }",
    "animate { target primitive 3 key 0 position 1 2 3 }",
    "light { kind point }\nanimate { target light 0 key 1 position 0 0 0 key 0.5 position 1 1 1 }",
    "light { kind laser }",
    "cascade { resolution 1 4 4 }",
    "lod_distances 10 5",
    "frobnicate 3",
    "camera { position 1 2",
    "camera position 1 2 3",
    "sky -1 0 0",
]


def main():
    out = []
    for text in SNIPPETS:
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "x.scene")
            with open(path, "w") as f:
                f.write(text)
            r = subprocess.run([EXE, "scene", path, os.path.join(tmp, "x.sdfs")], capture_output=True, text=True)
            msg = r.stderr.strip()
            assert r.returncode != 0 and msg.lower().startswith("error: "), (text, r.returncode, r.stdout, r.stderr)
            out.append({"text": text, "error": msg[len("error: "):]})
    with open(os.path.join(ROOT, "tests", "golden_parse_errors.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(len(out), "snippets")


if __name__ == "__main__":
    main()
