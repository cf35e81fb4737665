"""Quick check of the sharded (virtual shards) path vs the single engine."""
import sys
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
N, a, t = 1048351, 12345, 6
prob = shs.FactoringProblem.make(N, a, t)
o = shs.SimulatorOptions(qubit_ceiling=64, combine="exact", tiling="force")
single = shs.IterativeShorEngine(prob, shs.ErrorConfig(), o)
sh = shs.ShardedShorEngine.virtual(prob, shs.ErrorConfig(), o, nshards=2)
r = single.run(3, 0); s = sh.run(3, 0)
print("bits equal", r.bits.j == s.bits.j, [x.p1 for x in r.trace] == [x.p1 for x in s.trace], flush=True)
