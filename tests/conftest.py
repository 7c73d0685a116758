import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running statistical check")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(ROOT, "tests", "golden")
    out = {}
    for name in os.listdir(d):
        if name.endswith(".json"):
            with open(os.path.join(d, name)) as f:
                out[name[:-5]] = json.load(f)
    return out


@pytest.fixture(scope="session")
def parity_log():
    """Append one JSON record per parity comparison (exempt counts, fingerprint merges)
    to $LSH_PARITY_LOG (default gpurun_out/parity_log.jsonl) and echo it to stdout."""
    import json
    path = os.environ.get("LSH_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_log.jsonl"))
    os.makedirs(os.path.dirname(path), exist_ok=True)

    def log(rec: dict):
        line = json.dumps(rec, sort_keys=True)
        print("PARITY " + line)
        with open(path, "a") as f:
            f.write(line + "\n")
    return log
