"""Golden vectors for the tower trainer and the cost model, from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):
    python tests/golden/gen_golden_towers.py
Writes tests/golden/reference_towers.npz:
  ds_image / ds_text / W0_image / W0_text : `disco train` defaults (cli.py:227-240,
      336-343): generate_dataset(M=64, D_in=8, latent=4, noise=0.05, seed=0),
      init_tower_params(8, 4, seed=1), t = 20 (towers.py:36)
  traj_naive / traj_disco : train_run losses, 50 steps, batch 16, world 2, lr 0.2
      (towers.py:205-280); W_final_* : final weights of the naive run
  analytic : analytic_footprint rows for a (method, B, N, L, D, bytes) grid (costs.py:97-113)
  measured : measured_detail(mode, B, N, D) (costs.py:143-187) for a small grid
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from disco import costs, towers  # noqa: E402  (the reference package)


def main():
    out = {}
    ds = towers.generate_dataset(M=64, D_in=8, latent_dim=4, noise_scale=0.05, seed=0)
    p0 = towers.init_tower_params(8, 4, seed=1)
    out["ds_image"], out["ds_text"] = ds.image_inputs, ds.text_inputs
    out["W0_image"], out["W0_text"] = p0.W_image, p0.W_text
    out["t"] = np.array(p0.t)
    for mode, world in (("naive", 1), ("disco", 2)):
        p = p0.clone()
        traj = towers.train_run(towers.TrainConfig(global_batch=16, world_size=world, steps=50,
                                                   learning_rate=0.2, seed=0, mode=mode), ds, p)
        out[f"traj_{mode}"] = np.array([loss for _, loss in traj])
        out[f"W_final_{mode}_image"], out[f"W_final_{mode}_text"] = p.W_image, p.W_text
    rows = []
    for method in costs.METHODS:
        for B, N, L, D, bps in ((65536, 64, 12, 1024, 4), (32768, 8, 12, 512, 2 + 2), (1024, 2, 1, 512, 8),
                                (196608, 8, 24, 768, 4), (16, 16, 3, 5, 8)):
            r = costs.analytic_footprint(costs.CostInputs(B=B, N=N, L=L, D=D, bytes_per_scalar=bps), method)
            rows.append([costs.METHODS.index(method), B, N, L, D, bps, r.backbone_elements, r.loss_elements,
                         r.total_elements, r.loss_flops, r.bytes])
    out["analytic"] = np.array(rows, dtype=np.int64)
    meas = []
    for mode in ("naive", "disco"):
        for B, N, D in ((64, 1, 8), (64, 2, 8), (256, 4, 16), (256, 8, 16)):
            lp, lf, xp = costs.measured_detail(mode, B, N, D)
            meas.append([int(mode == "disco"), B, N, D, lp, lf, xp])
    out["measured"] = np.array(meas, dtype=np.int64)
    path = os.path.join(HERE, "reference_towers.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
