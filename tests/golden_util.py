import json
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).with_name("golden") / "reference_golden.json"
REFERENCE_SRC = Path("/root/reference/pkg/src")


@lru_cache(maxsize=1)
def golden() -> dict:
    return json.loads(GOLDEN.read_text())
