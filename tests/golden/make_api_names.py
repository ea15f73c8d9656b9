"""Record the reference's public API surface (function names of holopipe/api.py) as a fixture.

Run in the build container: python tests/golden/make_api_names.py"""
import ast
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
tree = ast.parse(open("/root/reference/pkg/src/holopipe/api.py").read())
names = sorted(n.name for n in tree.body if isinstance(n, ast.FunctionDef) and not n.name.startswith("_"))
json.dump({"source": "holopipe/api.py (public functions), extracted by tests/golden/make_api_names.py",
           "names": names}, open(os.path.join(HERE, "reference_api_names.json"), "w"), indent=1)
