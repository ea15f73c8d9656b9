"""Record the reference's public API surface (function names and parameter lists of holopipe/api.py)
as a fixture.  Run in the build container: python tests/golden/make_api_names.py"""
import ast
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
tree = ast.parse(open("/root/reference/pkg/src/holopipe/api.py").read())
funcs = [n for n in tree.body if isinstance(n, ast.FunctionDef) and not n.name.startswith("_")]


def params(fn):
    a = fn.args
    nd = len(a.args) - len(a.defaults)   # [name] or [name, default]
    return [[arg.arg] if i < nd else [arg.arg, ast.literal_eval(a.defaults[i - nd])] for i, arg in enumerate(a.args)]


json.dump({"source": "holopipe/api.py (public functions), extracted by tests/golden/make_api_names.py",
           "names": sorted(f.name for f in funcs),
           "params": {f.name: params(f) for f in sorted(funcs, key=lambda f: f.name)}},
          open(os.path.join(HERE, "reference_api_names.json"), "w"), indent=1)
