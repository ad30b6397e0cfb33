cd $GRAFT_REPO_ROOT
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import tests.test_gpu_engine as T
from paper_2604_16400_b200.layer import AdamWConfig
from paper_2604_16400_b200.backend import CudaLoraBackend, make_engine
from paper_2604_16400_b200.configs import CONFIGS
import coserve.engine as engine, coserve.domain as domain
for lr in (1e-3, 3e-4, 1e-4):
    sc = T._scenario(30.0)
    be = CudaLoraBackend(CONFIGS["tiny"], sorted(sc.stream_map), 4, families={s: c.family for s, c in sc.stream_map.items()}, optimizer=AdamWConfig(lr=lr), noise_every=5)
    be.calibrate(0.03)
    eng = make_engine(engine, be)(sc, 3)
    orig = eng._launcher_scan; forced = []
    def scan(eng=eng, orig=orig, forced=forced):
        if not forced:
            for rid in (1, 2, 3): eng.replicas[rid].set_state(domain.ReplicaState.IDLE, eng.now)
            forced.append(1)
        orig()
    eng._launcher_scan = scan
    led = eng.run()
    print(lr, [ (r["round_index"], round(r["mean_loss"],3), r["stopped"]) for r in led.fl_rounds][:12], "B:", [rep.batch_cfg for rep in eng.replicas.values()])
PY
