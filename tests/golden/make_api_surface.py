"""Record the reference's public API surface (names in cpfit.__all__, and for
every public callable its parameter names, kinds and defaults) as
tests/golden/api_surface.json.  Run here, where /root/reference exists:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_api_surface.py
tests/test_api_surface.py checks the drop-in package against it."""
import inspect
import json
import os

import cpfit

surface = {"all": sorted(cpfit.__all__), "signatures": {}}
for name in surface["all"]:
    obj = getattr(cpfit, name)
    if inspect.isclass(obj) or not callable(obj):
        continue
    surface["signatures"][name] = [
        [p.name, p.kind.name, None if p.default is inspect.Parameter.empty else repr(p.default)]
        for p in inspect.signature(obj).parameters.values()]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "api_surface.json")
json.dump(surface, open(out, "w"), indent=1, sort_keys=True)
print(out, len(surface["all"]), "names", len(surface["signatures"]), "signatures")
