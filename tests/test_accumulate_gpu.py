"""The fused combine of order sharding: fllf_apply_accumulate
adds each partial output into the destination with atomics, locally or into
another process's buffer mapped through CUDA IPC (dist.P2PCombine).  The
multi-process case runs 2 and 3 processes on ONE GPU (IPC between processes
works on a single device; no kernel waits on another -- the ranks only meet
at host barriers); on a multi-GPU node the same code adds over NVLink."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import fllf_oracle as O
from paper_2206_04681_b200 import synth

pytestmark = pytest.mark.gpu
TOL_OUT = 2e-3


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


@pytest.mark.parametrize("H,W,B", [(77, 90, 1), (64, 96, 2), (45, 70, 1)])
def test_partials_accumulate_to_full(F, H, W, B):
    levels, K, T, sig, m = 4, 9, 510.0, 25.0, 2.0
    frames = np.stack([synth.uniform_image(H, W, seed=70 + b) for b in range(B)]).astype(np.float32)
    d = torch.from_numpy(frames).cuda()
    out = torch.zeros_like(d)
    for kb, ke, base in ((1, 4, True), (4, 7, False), (7, 10, False)):
        with F.Plan(H, W, levels, K, T, sig, m, batch=B, k_begin=kb, k_end=ke, include_base=base) as p:
            p.build(d)
            F.fllf_apply_accumulate(p.handle, out)
            torch.cuda.synchronize()
    for b in range(B):
        ref = O.fourier_llf(frames[b].astype(np.float64), levels, K, T, sig, m)
        assert np.abs(out[b].cpu().numpy() - ref).max() <= TOL_OUT


def test_accumulate_errors(F):
    d = torch.rand(64, 64, device="cuda")
    o = torch.zeros_like(d)
    with F.Plan(64, 64, 3, 4) as p:
        p.build(d)
        args = F.fllf_apply_args()
        args.mode = F.FLLF_MAPS  # the C boundary itself refuses MAPS
        st = F.lib.fllf_apply_accumulate(p.handle, ctypes.byref(args), o.data_ptr(), 64 * 4, None)
        assert st == F.FLLF_ERR_INVALID_ARGUMENT
    with pytest.raises(F.FllfError):
        F.ipc_open(b"\0" * F.IPC_HANDLE_BYTES)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rgb, params, path):
    import torch.distributed as dist

    from paper_2206_04681_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    levels, K, T, sig, m = params
    img = torch.from_numpy(rgb).cuda()
    comb = D.P2PCombine(img, levels, K, T, sig, m)
    for _ in range(2):  # the buffer and the mappings are reused across calls
        out = comb.run()
    if rank == 0:
        np.save(path, out.cpu().numpy())
    comb.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_combine_processes(F, tmp_path, world):
    C, H, W = 3, 52, 83
    rgb = np.stack([synth.uniform_image(H, W, seed=90 + c) for c in range(C)]).astype(np.float32)
    params = (4, 10, 510.0, 20.0, 2.0)
    path = str(tmp_path / "out.npy")
    mp.spawn(_worker, args=(world, _free_port(), rgb, params, path), nprocs=world, join=True)
    got = np.load(path)
    for c in range(C):
        ref = O.fourier_llf(rgb[c].astype(np.float64), *params)
        assert np.abs(got[c] - ref).max() <= TOL_OUT
