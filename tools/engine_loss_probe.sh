cd $GRAFT_REPO_ROOT
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import tests.test_gpu_engine as T
from paper_2604_16400_b200.layer import AdamWConfig
from paper_2604_16400_b200.backend import CudaLoraBackend, make_engine
from paper_2604_16400_b200.configs import CONFIGS
import coserve.engine as engine, coserve.domain as domain
sc = T._scenario(30.0)
be = CudaLoraBackend(CONFIGS["tiny"], sorted(sc.stream_map), 4, families={s: c.family for s, c in sc.stream_map.items()}, optimizer=AdamWConfig(lr=1e-3), noise_every=5)
be.calibrate(0.03)
log = []
ots, oag = be.train_step, be.aggregate
def ts(replica, B, b, now):
    r = ots(replica, B, b, now)
    log.append(("step", replica.id, B, b, round(be._losses[replica.id], 3), be._cursor))
    return r
def ag(f, rep):
    log.append(("AGG", rep, [round(float(be.stack.trainers[("replica", r)].flat_master.norm()), 4) for r in rep]))
    oag(f, rep)
    log.append(("AGG-after", [round(float(be.stack.trainers[("replica", r)].flat_master.norm()), 4) for r in rep]))
be.train_step, be.aggregate = ts, ag
eng = make_engine(engine, be)(sc, 3)
orig = eng._launcher_scan; forced = []
def scan():
    if not forced:
        for rid in (1, 2, 3): eng.replicas[rid].set_state(domain.ReplicaState.IDLE, eng.now)
        forced.append(1)
    orig()
eng._launcher_scan = scan
led = eng.run()
for e in log: print(e)
PY
