"""Generate `tests/golden/acceptance.npz`: the reference's own acceptance suites
(pkg/src/gradcomp/verify.py) and degenerate Gram-Schmidt cases, recorded from
the REFERENCE ITSELF so the GPU tests can be checked against it.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_acceptance.py

Recorded:
* warmstart (verify.py:41-96): the 20 seeded 64x48 gapped matrices
  (`_gap_matrix`), the reference's best rank-2 error of each
  (`reconstruction_error(m, best_rank_r(m, 2, seed=1))`) and the iteration at
  which the reference's PowerSGD reached it;
* linearity (verify.py:99-143): the conditioned least-squares instance
  (problems.py:53-116, seed 3, spectrum (10, 5, 2)) and the final parameters of
  the reference's W=4 and W=1 runs after 200 steps (run_training);
* orthogonalize with repeated degenerate draws (linalg.py:82-88): inputs whose
  attempt-0 (and attempt-1) replacement columns are themselves degenerate, and
  the reference's outputs.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from gradcomp import verify  # noqa: E402
from gradcomp.comm import Communicator  # noqa: E402
from gradcomp.compressors import CompressionContext, make_compressor  # noqa: E402
from gradcomp.linalg import _replacement_column, best_rank_r, orthogonalize, reconstruction_error  # noqa: E402
from gradcomp.train import run_training  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    # ---- warmstart
    mats, errs, reached = [], [], []
    for s in range(verify.WARMSTART_MATRICES):
        m = verify._gap_matrix(s)
        mats.append(m)
        oracle_err = reconstruction_error(m, best_rank_r(m, 2, seed=1))
        errs.append(oracle_err)
        comp = make_compressor("powersgd", 2)
        comm = Communicator(1)
        hit = -1
        for it in range(1, verify.WARMSTART_ITER_LIMIT + 1):
            trip = comp.round_trip([m], CompressionContext(7, 0, it), comm)
            err = float(np.linalg.norm(m - trip.aggregated))
            if abs(err - oracle_err) <= verify.WARMSTART_REL_TOL * oracle_err:
                hit = it
                break
        reached.append(hit)
    out["ws_mats"] = np.stack(mats)
    out["ws_best_err"] = np.array(errs)
    out["ws_reached"] = np.array(reached)
    # ---- linearity
    prob = verify._linearity_problem()
    out["lin_inputs"] = prob.inputs
    out["lin_targets"] = prob.targets
    multi = run_training(verify._linearity_config(verify.LINEARITY_WORKERS), problem=verify._linearity_problem())
    single = run_training(verify._linearity_config(1), problem=verify._linearity_problem())
    for k, p in enumerate(multi.final_params):
        out[f"lin_w4_p{k}"] = p
    for k, p in enumerate(single.final_params):
        out[f"lin_w1_p{k}"] = p
    out["lin_w4_loss"] = np.array([r.loss for r in multi.records])
    out["lin_w1_loss"] = np.array([r.loss for r in single.records])
    # ---- orthogonalize: repeated degenerate draws
    cases = {}
    n = 5  # column 1 = 0; column 0 = the attempt-0 draw for column 1 -> attempt 1
    cases["attempt1"] = np.stack([_replacement_column(n, 1, 0), np.zeros(n)], axis=1)
    n = 6  # column 2 = 0; columns 0, 1 span the attempt-0 and attempt-1 draws for column 2 -> attempt 2
    cases["attempt2"] = np.stack([_replacement_column(n, 2, 0), _replacement_column(n, 2, 1), np.zeros(n)], axis=1)
    n = 4  # every column zero: one replacement per column
    cases["zeros4"] = np.zeros((n, 3))
    for k, v in cases.items():
        out[f"orth_in_{k}"] = v
        out[f"orth_out_{k}"] = orthogonalize(v)
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **out)
    print("wrote acceptance.npz:", len(out), "arrays; warmstart reached", reached)


if __name__ == "__main__":
    main()
