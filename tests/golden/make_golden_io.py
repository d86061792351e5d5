"""Record the reference loader's outcome for every corpus file
(tests/golden/io_cases.json).  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py
"""
import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import blk.io  # noqa: E402
from io_corpus import CASES  # noqa: E402
from test_io import _outcome  # noqa: E402

out = {}
with tempfile.TemporaryDirectory() as d:
    for name, content in sorted(CASES.items()):
        p = Path(d) / f"{name}.musr"
        p.write_bytes(content.encode("utf-8"))
        out[name] = _outcome(blk.io.load_musr_data, p)
(HERE / "io_cases.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
print(f"{len(out)} cases")
