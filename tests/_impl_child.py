"""Child process for test_gpu_parity.test_sweep_impl_parity: config 5
reduced (16^2, p=6, one BE step) under the IHDG_SWEEP_IMPL of the environment
(the kernel choice is read once per process), checked against the oracle."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1711_01175_b200.iteration import IterationConfig, run_time_dependent
    from paper_1711_01175_b200.workloads import make_config
    from tests.oracle_bridge import oracle_initial, oracle_solver, rel_l2

    torch.cuda.set_device(0)
    wl = make_config(5, seed=0, cells=16, kappa=float(sys.argv[1]), n_steps=1)
    reps = run_time_dependent(wl.mesh, wl.problem, wl.ops, IterationConfig(tol=1e-10), wl.dt,
                              n_steps=1, initial=wl.initial, keep_states=True)
    S = oracle_solver(wl)
    _, refs = S.run_time_dependent(oracle_initial(wl, S), 1, tol=1e-10)
    its = [r.iterations for r in reps], [r["iterations"] for r in refs]
    err = max(rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) for r, o in zip(reps, refs))
    print(f"{os.environ.get('IHDG_SWEEP_IMPL', 'default')}: iterations {its[0]} vs {its[1]}, rel L2 {err:.2e}")
    assert its[0] == its[1] and err < 1e-10


if __name__ == "__main__":
    main()
