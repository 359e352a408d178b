"""Device-memory plumbing: numpy <-> torch CUDA buffers for the C ABI.

PyTorch is used only for device allocation, streams and copies; all
arithmetic on the hot path happens in libconcpd_b200.so kernels.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def torch_mod():
    return _lib.require_cuda()


def device():
    torch = torch_mod()
    return torch.device("cuda", torch.cuda.current_device())


def to_dev_f64(a):
    """Upload a numpy matrix (row-major) as a contiguous fp64 CUDA tensor."""
    torch = torch_mod()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def tensor_to_dev(t, dtype="fp64"):
    """Upload a tensor in first-index-fastest (Fortran) physical order.

    numpy arrays of any layout are converted (a Fortran-contiguous array is
    copied without reordering).  torch CUDA tensors are accepted as given if
    their memory is already Fortran-ordered for their logical shape.
    Returns (flat CUDA tensor, dims tuple).
    """
    torch = torch_mod()
    want = torch.float64 if dtype == "fp64" else torch.float32
    if isinstance(t, torch.Tensor):
        dims = tuple(int(d) for d in t.shape)
        if t.is_cuda and t.dtype == want and tuple(t.stride()) == fortran_strides(dims):
            return t.as_strided((t.numel(),), (1,)), dims      # already first-index-fastest
        if not t.is_cuda and t.dtype == want and tuple(t.stride()) == fortran_strides(dims):
            # host buffer already first-index-fastest (pinned: asynchronous DMA)
            flat = t.as_strided((t.numel(),), (1,))
            return flat.to(device=device(), non_blocking=t.is_pinned()), dims
        # any other layout: copy as stored (one contiguous DMA when the memory
        # is dense), reorder on the device
        perm = tuple(range(t.ndim - 1, -1, -1))
        if t.is_cuda or not t.is_contiguous():
            flat = t.permute(*perm).contiguous().reshape(-1)   # Fortran order of t
            return flat.to(device=device(), dtype=want), dims
        dev = t.to(device=device())
        return dev.permute(*perm).contiguous().reshape(-1).to(want), dims
    a = np.asarray(t)
    dims = tuple(int(d) for d in a.shape)
    np_dtype = np.float64 if dtype == "fp64" else np.float32
    a = np.asarray(a, dtype=np_dtype)
    if a.flags.f_contiguous or a.ndim <= 1:
        flat = np.ravel(a, order="F")          # a view: no host copy
        return torch.from_numpy(np.ascontiguousarray(flat)).to(device()), dims
    # C-ordered (numpy's default) or strided: a host-side reorder of a 400^3
    # block takes ~0.2 s; upload the dense bytes and permute on the device
    dev = torch.from_numpy(np.ascontiguousarray(a)).to(device())
    perm = tuple(range(a.ndim - 1, -1, -1))
    return dev.permute(*perm).contiguous().reshape(-1), dims


def source_dtype(t):
    """"fp32" for float32 input (numpy or torch), else "fp64" (the
    reference casts everything else to float64, solver.py:91)."""
    dt = getattr(t, "dtype", None)
    if dt is None:
        return "fp64"
    torch = torch_mod()
    return "fp32" if dt in (np.float32, torch.float32) else "fp64"


def cast_flat(flat, dtype):
    """Device-side cast of a flat buffer to the solve precision."""
    torch = torch_mod()
    return flat.to(torch.float64 if dtype == "fp64" else torch.float32)


def fortran_strides(dims):
    st, acc = [], 1
    for d in dims:
        st.append(acc)
        acc *= int(d)
    return tuple(st)


def fortran_view(flat, dims):
    """Logical-shape view of a flat first-index-fastest CUDA buffer."""
    return flat.as_strided(tuple(int(d) for d in dims), fortran_strides(dims))


def ptr(x):
    return x.data_ptr()


def stream():
    return _lib.stream_handle()


def to_host(x):
    return x.detach().cpu().numpy()
