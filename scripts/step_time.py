import sys, time
sys.path.insert(0, '.')
import paper_2308_05047_b200 as shs
import torch
eng = shs.IterativeShorEngine(shs.FactoringProblem.make(4294967213, 5), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
eng.set_orbit(sys.argv[1] == '1')
eng.state_init()
prefix = 0
err = shs.ErrorConfig()
for s in range(0, 12):
    t0 = time.perf_counter()
    p0, p1 = eng.stage_probs(s, prefix)
    t1 = time.perf_counter()
    m = shs.sample_measurement(p1, 2308, 0, s, err)
    b = m["sampled_bit"]
    t2 = time.perf_counter()
    eng.stage_collapse(b, p1 if b else p0)
    t3 = time.perf_counter()
    prefix |= b << s
    print(s, f"probs {1e3*(t1-t0):.2f} sample {1e3*(t2-t1):.2f} collapse {1e3*(t3-t2):.2f} bit {b}", flush=True)
