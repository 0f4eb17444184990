import sys, time, warnings, cProfile, pstats
sys.path.insert(0, '.')
import torch
from bench import detector_params
from paper_1901_07306_b200 import DetectorState
from tools.workloads import CONFIG2, generate
h, o, s = generate(CONFIG2, "torch", torch.device("cuda", 0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    st = DetectorState.create(detector_params())
st.process_batch(h, o); torch.cuda.synchronize()
for _ in range(3): st.finalize_window()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): r = st.finalize_window()
torch.cuda.synchronize()
print("finalize ms", (time.perf_counter() - t) / 20 * 1e3, len(r))
t = time.perf_counter()
for _ in range(20): st.seav.clear(); st.ldca.clear()
torch.cuda.synchronize()
print("reset ms", (time.perf_counter() - t) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): st.finalize_window()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
