cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in cfg5 cfg2 n8192; do
TAG=default timeout -s KILL 300 python tools/time_step.py $c >> gpurun_out/steps.log 2>&1
TAG=big BD_BIG_MIN_N=4000 timeout -s KILL 300 python tools/time_step.py $c >> gpurun_out/steps.log 2>&1
done
cat > /tmp/cfg4.py <<'PY'
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1703_02484_b200.core import CounterRng, ParticleSystem, PeriodicBox, SimParams, box_length_for_density
from paper_1703_02484_b200.dynamics import LongRangeSimulation
from paper_1703_02484_b200.initial import InitConfig, init_arrays
from paper_1703_02484_b200.triangulation import build_initial
n=1<<20; box=PeriodicBox(box_length_for_density(n,1.0,0.6))
pos,t,a,m=init_arrays(InitConfig(n=n,box=box,sigma=1.0,types=[(0.5,3.0,3.0),(0.5,-3.0,-1.5)],seed=1))
sys_=ParticleSystem(pos,t,a,m,box); tri=build_initial(sys_.positions,box,method="device")
sim=LongRangeSimulation(sys_,SimParams(n=n,sigma=1.0,dt=0.01,diffusion=0.01,r_cutoff=2.5),CounterRng(1,2),tri=tri,force="short-range")
sim.run(5); st=sim.run(15)
print("cfg4", os.environ.get("TAG"), np.mean([s.step_ms for s in st]))
PY
TAG=default timeout -s KILL 300 python /tmp/cfg4.py >> gpurun_out/steps.log 2>&1
TAG=big0 BD_BIG_MIN_N=0 timeout -s KILL 300 python /tmp/cfg4.py >> gpurun_out/steps.log 2>&1
cat gpurun_out/steps.log
