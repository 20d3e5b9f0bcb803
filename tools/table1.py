"""Table 1-style statistics: mean #Recurrence (RAC passes per
assignment, GPU rac_search) and mean #Revision (AC-3 revisions per assignment, CPU oracle
search over the same tree) over the first K assignments of Alg. 2 backtracking search.

The paper's instances, domain size and tightness are unpublished; here d = 20 and the
tightness is each cell's phase-transition estimate t_cr = 1 - d^(-2/(p(n-1))) (so search
does not end at the root), seed 1.  Trends, not values, are comparable.
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

PAPER = {  # (n, density): (#Revision, #Recurrence) -- PAPER.md lines 261-285
    (100, .1): (307.6, 4.509), (100, .25): (626.4, 4.103), (100, .5): (965.2, 3.752), (100, .75): (1612.4, 3.573),
    (100, 1.): (2714.1, 3.462), (250, .1): (1152.0, 4.804), (250, .25): (2532.6, 4.167), (250, .5): (4629.6, 3.794),
    (250, .75): (7881.9, 3.617), (250, 1.): (12405.6, 3.441), (500, .1): (3250.9, 4.620), (500, .25): (7619.8, 4.126),
    (500, .5): (18793.8, 3.952), (500, .75): (28218.4, 3.728), (500, 1.): (42557.7, 3.455),
    (750, .1): (6195.7, 4.766), (750, .25): (13768.6, 4.020), (750, .5): (36220.6, 3.940),
    (750, .75): (61171.7, 3.703), (750, 1.): (71509.8, 3.597), (1000, .1): (8322.2, 4.831),
    (1000, .25): (24544.3, 4.381), (1000, .5): (39707.7, 4.048), (1000, .75): (65446.2, 3.755),
    (1000, 1.): (107680.5, 3.556)}


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    ns = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["100", "250", "500", "750", "1000"])]
    with_ac3 = "--ac3" in sys.argv
    d = 20
    rows = []
    for n in ns:
        for p in (0.1, 0.25, 0.5, 0.75, 1.0):
            t = 1.0 - d ** (-2.0 / (p * (n - 1)))
            ctx = rac.RacContext.create_random(n, d, synth.quant_density(p), synth.quant_tightness(t), 1)
            full = synth.full_domains(np.full(n, d))
            t0 = time.time()
            r, sol, st = ctx.search(full, max_assignments=K)
            wall = time.time() - t0
            a = max(st["assignments"], 1)
            row = {"n": n, "density": p, "d": d, "tightness": round(t, 5), "result": {0: "solution", 1: "unsat", 2: "budget"}[r],
                   "assignments": st["assignments"], "recurrence_per_assignment": st["recurrences"] / a,
                   "wipeout_frac": st["wipeouts"] / a, "us_per_assignment_gpu": st["enforce_seconds"] / a * 1e6,
                   "root_iterations": st["root_iterations"], "paper_recurrence": PAPER[(n, p)][1],
                   "paper_revision": PAPER[(n, p)][0], "search_wall_s": round(wall, 3)}
            if with_ac3 and n <= 250:
                import oracle
                inst = synth.random_csp(n, d, p, t, 1)
                orc = oracle.Oracle.from_instance(inst)
                ro, _, so = orc.search(full, max_assignments=min(K, 300), engine="ac3")
                row["revision_per_assignment_ac3"] = so["recurrences"] / max(so["assignments"], 1)
                row["ac3_assignments"] = so["assignments"]
            rows.append(row)
            print(json.dumps(row), flush=True)
    json.dump(rows, open("gpurun_out/table1.json", "w"), indent=1)


if __name__ == "__main__":
    main()
