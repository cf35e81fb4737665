import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "ms/stage %.2f" % d["ms_per_step"], "stage frac %.3f" % d["stage_frac_of_hbm"],
              {k: (round(v["avg_ms"], 3), v["achieved_gbs"] and round(v["achieved_gbs"])) for k, v in d["kernels"].items()},
              "s/run %.2f (dense %.2f)" % (d["s_per_run"], d.get("s_per_run_dense", 0)), "e2e %.3g" % d["e2e"]["value"], d["clocks"],
              "cpu", d.get("cpu_baseline", {}).get("value"),
              {k: (round(v["runs_per_s"]), round(v.get("reference_cpu_runs_per_s_1core", 0)))
               for k, v in d.get("batched_small_n", {}).items()})
    except Exception as e:
        print(f, "ERR", e)
