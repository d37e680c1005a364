import cProfile, pstats, sys, copy
sys.path.insert(0, '/root/repo/profiles'); sys.path.insert(0, '/root/repo')
import numpy as np
import dropin_jitter as DJ
from paper_2510_18855_b200 import objective as O
rng = np.random.default_rng(0)
S, T, nf, V = 8, 512, 1024, 32768
w = rng.normal(0.0, 0.8, (nf, V))
task = DJ.Task(prompt_id=17)
rollouts = []
for _ in range(S):
    lp = rng.normal(-10.4, 0.3, T); inf = lp - rng.normal(0, 0.233, T)
    rollouts.append(DJ.Rollout([O.TokenRecord(int(y), float(b), float(a), float(a), 0) for y, a, b in zip(rng.integers(0, V, T), lp, inf)]))
rewards = [float(x) for x in rng.integers(0, 2, S)]
groups = [O.PromptGroup(task=task, rollouts=rollouts, rewards=rewards, advantages=list(O.group_advantages(rewards)))]
theta = DJ.Params(w); cfg, bounds = O.ObjectiveConfig(), O.MaskingBounds()
buf = np.empty_like(w)
for _ in range(3): O.objective_and_grad(copy.deepcopy(groups), theta, theta, None, cfg, bounds, precision="bf16", grad_out=buf)
gs = [copy.deepcopy(groups) for _ in range(20)]
pr = cProfile.Profile(); pr.enable()
for g in gs: O.objective_and_grad(g, theta, theta, None, cfg, bounds, precision="bf16", grad_out=buf)
pr.disable()
st = pstats.Stats(pr); st.sort_stats('tottime').print_stats(18)
