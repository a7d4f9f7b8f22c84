"""Decode-step and 72-row verify latency of any registered shape against its
HBM floor (weights streamed once per pass):

    python tools/shape_time.py mistral-7b
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from paper_2506_15556_b200.shapes import SHAPES  # noqa: E402

for name in sys.argv[1:] or ["mistral-7b"]:
    print(json.dumps(bench.pass_latency(SHAPES[name], 6533.2)))
