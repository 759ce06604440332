"""Host logic of the measurement tools (no GPU): the FER sweep's checkpoint/resume keys."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_fer_sweep_resume_keys(tmp_path):
    import fer_sweep as fs

    out = tmp_path / "fer.jsonl"
    rows = [{"code": [32768, 27568], "design_ebn0": 4.0, "ebn0": 3.5, "profile": "i8", "frames": 10},
            {"code": [32768, 27568], "design_ebn0": 4.0, "ebn0": 4.5, "profile": "f32", "first_frame": 100,
             "frames": 50, "max_frames": 50}]
    out.write_text("\n".join(json.dumps(r) for r in rows) + "\nnot json\n")
    done = fs.completed(str(out))
    assert ((32768, 27568), 4.0, 3.5, "i8") in done
    assert ((32768, 27568), 4.0, 4.5, "f32", 100, 50) in done
    assert ((32768, 27568), 4.0, 3.75, "i8") not in done
    fs._OUT = str(out)
    fs.emit({"code": [2048, 1723], "design_ebn0": 4.0, "ebn0": 4.0, "profile": "i8", "frames": 1})
    assert ((2048, 1723), 4.0, 4.0, "i8") in fs.completed(str(out))
    fs._OUT = None
