import os, subprocess, sys, numpy as np
code = ("import sys; sys.path.insert(0, '.'); import numpy as np\n"
    "import paper_1607_00968_b200 as hz; from paper_1607_00968_b200 import configs\n"
    "nl = int(sys.argv[2]); kind = sys.argv[3]\n"
    "cfg = configs.config2(nlevels=nl, k=8, nx=257, nz=129); cfg.precond_precision = 'c64'; cfg.cycle = kind\n"
    "o = hz.HelmholtzSolveOptions.from_config(cfg); o.cycle.pre = int(sys.argv[4]); o.cycle.post = int(sys.argv[5])\n"
    "S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), o)\n"
    "b = configs.random_block(cfg.num_nodes, 8, seed=11)\n"
    "np.save(sys.argv[1], S.cycle(b))\n")
def run(path, env, *a):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code, path, *a], env=e, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-1500:]
    return np.load(path)
for nl, pre, post in ((3, 1, 0), (3, 0, 1), (3, 2, 2), (4, 2, 2)):
    a = run("/tmp/a.npy", {"HZ_S9_MIN_NODES": "0"}, str(nl), "V", str(pre), str(post))
    b = run("/tmp/b.npy", {"HZ_S9": "0"}, str(nl), "V", str(pre), str(post))
    d = np.abs(a - b)
    print(nl, pre, post, "equal" if np.array_equal(a, b) else f"maxdiff {d.max():.3e} rel {np.linalg.norm(a-b)/np.linalg.norm(b):.3e} nbad {np.count_nonzero(d)} first {np.argwhere(d > 0)[:3].tolist()}")
