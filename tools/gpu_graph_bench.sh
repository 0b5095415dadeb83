timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "graph or full_step" 2>&1 | tail -3
for G in 1 0; do
python - << PY
import sys, json
sys.argv = ["bench.py"]
import bench, paper_2102_13133_b200 as pic
orig = pic.Context.__init__
def init(self, *a, **k):
    orig(self, *a, **k)
    self._set_graphs(bool($G))
pic.Context.__init__ = init
sys.argv = ["bench.py", "--config", "thermal", "--steps", "50", "--warmup", "5", "--no-e2e", "--no-cpu-baseline"]
bench.main()
PY
done
