"""Writes tests/golden/reference_api.json: the reference package's public names
(drgraph.__all__, pkg/src/drgraph/__init__.py:57-70) and the parameter lists of its
callables, read by importing the reference in the build container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_api_golden.py
"""
import inspect
import json
import os

import drgraph

out = {"__all__": list(drgraph.__all__), "params": {}}
for name in drgraph.__all__:
    obj = getattr(drgraph, name)
    if callable(obj) and not inspect.isclass(obj):
        out["params"][name] = [p.name for p in inspect.signature(obj).parameters.values()]
    elif inspect.isclass(obj) and hasattr(obj, "__dataclass_fields__"):
        out["params"][name] = list(obj.__dataclass_fields__)
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_api.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(path, len(out["__all__"]), "names")
