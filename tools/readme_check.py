"""Run README.md's quick-start snippet at 32^3 on the GPU (documentation check)."""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
code = re.search(r"```python\n(.*?)```", open(os.path.join(ROOT, "README.md")).read(), re.S).group(1)
code = code.replace("n, nt = 256, 4", "n, nt = 32, 4")
env = {}
exec(compile(code, "README.md", "exec"), env)
print("readme snippet ok:", {k: float(env[k].norm()) for k in ("Hvt", "z", "g", "dv")})
