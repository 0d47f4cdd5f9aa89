import cProfile, pstats, sys, time, dataclasses
sys.path.insert(0, '.')
import bench
from paper_2102_05297_b200 import harness
ds, spec = bench.workload()
spec = dataclasses.replace(spec, repetitions=1000)
for _ in range(3): harness.simulate(spec, devices=[0])
import torch; torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10): harness.simulate(spec, devices=[0])
print("simulate ms", (time.perf_counter()-t)/10*1e3)
pr=cProfile.Profile(); pr.enable()
for _ in range(10): harness.simulate(spec, devices=[0])
pr.disable()
pstats.Stats(pr).sort_stats('cumtime').print_stats(25)
