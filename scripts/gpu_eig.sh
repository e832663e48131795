set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "syev or svqb or eig" > gpurun_out/pytest_eig.log 2>&1; echo "eig tests rc=$?"; tail -25 gpurun_out/pytest_eig.log
python - <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, ".")
from paper_2111_06552_b200 import device as D
dev = D.default_context()
for m in (16, 20, 40, 64, 65, 120, 160, 200, 232, 233, 400):
    a = np.random.default_rng(m).standard_normal((m, m)); a = (a + a.T) / 2
    A = torch.from_numpy(a).to(dev.device); w = dev.empty(m); v = dev.empty(m, m)
    for _ in range(3): D.syev(dev, A, w, v)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    for _ in range(10): D.syev(dev, A, w, v)
    e1.record(dev.stream); torch.cuda.synchronize()
    print(f"syev m={m}: {e0.elapsed_time(e1) / 10 * 1e3:8.1f} us", flush=True)
PY
