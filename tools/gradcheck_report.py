import sys; sys.path.insert(0, '.')
from paper_2605_05876_b200 import gradcheck
rep = gradcheck.run_gradcheck(n_scenes=20, seed=0)
print({k: rep[k] for k in ("total", "checked", "passed", "failed", "unstable")}, rep["per_class"])
for f in rep["failures"]:
    print(f["scene"], f["param"], f["index"], "a=%.6g fd=%.6g err=%.3g tol=%.3g h=%.2g" % (f["analytic"], f["fd"], f["error"], f["tol"], f["step"]))
