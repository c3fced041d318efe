"""Write-through host views of device tensors.

The reference exposes its state as live numpy arrays and mutates them in
place (`sys.positions[...] = x`, core.py:251, dynamics.py:93/130;
`abp.angles[i] = v`; the tests corrupt `tri.edge_tri[e, 0]`).  Here the
state lives in HBM, so reading an attribute returns a host copy.  A
HostView is that copy with the writes sent back: item assignment, in-place
operators and ufuncs with `out=` on the view (or on any slice of it) upload
the whole array to its tensor.  Copies made from a view are plain arrays.

A view records the owner's version when it is read; the owner bumps the
version whenever device code may have changed the tensor (a step, an op).
Writing through a view that is older than the device state raises instead
of overwriting newer device data with stale host data.
"""

from __future__ import annotations

import numpy as np


class StaleViewError(RuntimeError):
    pass


class Versioned:
    """Mixin: a device-state version counter for HostView staleness checks."""

    _bd_version = 0

    def bump_version(self):
        self._bd_version = self._bd_version + 1


class HostView(np.ndarray):
    """numpy copy of `tensor` whose in-place writes are uploaded to it."""

    def __new__(cls, tensor, owner: Versioned | None = None, name: str = "array"):
        arr = np.ascontiguousarray(tensor.detach().cpu().numpy()).view(cls)
        arr._bd_tensor = tensor
        arr._bd_owner = owner
        arr._bd_version = owner._bd_version if owner is not None else 0
        arr._bd_name = name
        arr._bd_root = arr
        return arr

    def __array_finalize__(self, obj):
        root = getattr(obj, "_bd_root", None)
        # slices / reshapes of the view stay bound to the device array; copies do not
        if root is not None and np.may_share_memory(self, root):
            self._bd_root = root
        else:
            self._bd_root = None

    def _bd_sync(self):
        root = getattr(self, "_bd_root", None)
        if root is None:
            return
        owner = root._bd_owner
        if owner is not None and owner._bd_version != root._bd_version:
            raise StaleViewError(
                f"{root._bd_name}: this host copy was read before the device state changed (a step or an op ran "
                f"since); read the attribute again and write through the fresh copy")
        import torch
        root._bd_tensor.copy_(torch.from_numpy(np.asarray(root)))

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._bd_sync()

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kwargs):
        args = [np.asarray(x) if isinstance(x, HostView) else x for x in inputs]
        views = []
        if out is not None:
            outs = []
            for o in out:
                if isinstance(o, HostView):
                    views.append(o)
                    outs.append(np.asarray(o))
                else:
                    outs.append(o)
            kwargs["out"] = tuple(outs)
        res = getattr(ufunc, method)(*args, **kwargs)
        for v in views:
            v._bd_sync()
        if out is not None and len(out) == 1 and isinstance(out[0], HostView):
            return out[0]
        return res

    def __array_function__(self, func, types, args, kwargs):
        plain = tuple(np.asarray(a) if isinstance(a, HostView) else a for a in args)
        res = func(*plain, **kwargs)
        if func in (np.copyto, np.put, np.place, np.putmask, np.fill_diagonal) and isinstance(args[0], HostView):
            args[0]._bd_sync()
        return res

    def fill(self, value):
        super().fill(value)
        self._bd_sync()

    def __reduce__(self):  # pickles as a plain array
        return np.asarray(self).copy().__reduce__()
