"""views/s of bench.run_config on the given BASELINE configs (default 3), one
JSON line each (run from a repo root; build first)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402

for cfg in (int(c) for c in (sys.argv[1:] or ["3"])):
    print(json.dumps({"config": cfg, **bench.run_config(cfg)}), flush=True)
