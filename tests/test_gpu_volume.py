"""Per-volume acceleration data built on the device (csrc/vdi_volume.cu):
brick maxima (vdi_volume_brick_max, the empty-space-skipping bound of the
samplers) and corner records (vdi_volume_cells), against numpy restatements,
for the vectorised u8 kernels (x extent a multiple of 8 / 4) and the generic
ones. Both feed exact generation: a brick maximum below a voxel it covers
would skip visible samples, a wrong corner would change a sample's bits.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2206_08660_b200 import device as dv  # noqa: E402

SHAPES = [(64, 40, 24), (72, 33, 17), (30, 21, 9), (8, 8, 8), (16, 9, 2)]  # (nx, ny, nz), each >= 2


def _volume(dims, dtype, seed):
    nx, ny, nz = dims
    rng = np.random.default_rng(seed)
    if dtype == "f32":
        a = rng.random((nz, ny, nx), dtype=np.float32)
    else:
        hi = 256 if dtype == "u8" else 65536
        a = rng.integers(0, hi, (nz, ny, nx)).astype(np.uint8 if dtype == "u8" else np.uint16)
    # sparse content: most bricks empty, as in the configs
    a[rng.random((nz, ny, nx)) < 0.9] = 0
    return a


def _brick_max_ref(a, log2=dv.BRICK_LOG2):
    nz, ny, nx = a.shape
    b = 1 << log2
    out = np.zeros(((nz + b - 1) // b, (ny + b - 1) // b, (nx + b - 1) // b), a.dtype)
    for bz in range(out.shape[0]):
        for by in range(out.shape[1]):
            for bx in range(out.shape[2]):
                # the brick plus one voxel of overlap (trilinear neighbours)
                out[bz, by, bx] = a[bz * b:min(bz * b + b, nz - 1) + 1,
                                    by * b:min(by * b + b, ny - 1) + 1,
                                    bx * b:min(bx * b + b, nx - 1) + 1].max()
    return out


@pytest.mark.parametrize("dims", SHAPES)
@pytest.mark.parametrize("dtype", ["u8", "u16", "f32"])
def test_brick_max(dims, dtype):
    a = _volume(dims, dtype, 7 * dims[0] + 3 * dims[1] + dims[2] + len(dtype))
    # u16 travels as int16 (same bits; the kernel reads raw voxels)
    vd = torch.from_numpy(a.view(np.int16) if dtype == "u16" else a).cuda()
    out = dv.alloc_bricks(vd, dims)
    dv.launch_bricks(vd, dtype, dims, out)
    got = out.cpu().numpy()
    ref = _brick_max_ref(a)
    np.testing.assert_array_equal(got.view(ref.dtype), ref)


@pytest.mark.parametrize("dims", SHAPES)
def test_cells_u8(dims):
    a = _volume(dims, "u8", 7)
    nx, ny, nz = dims
    vd = torch.from_numpy(a).cuda()
    out = dv.alloc_cells("u8", dims)
    dv.launch_cells(vd, "u8", dims, out)
    got = out.cpu().numpy()[:nx * ny * nz * 8].reshape(nz, ny, nx, 8)
    x1 = np.minimum(np.arange(nx) + 1, nx - 1)
    y1 = np.minimum(np.arange(ny) + 1, ny - 1)
    z1 = np.minimum(np.arange(nz) + 1, nz - 1)
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    corners = [(zz, yy, xx), (zz, yy, x1[xx]), (zz, y1[yy], xx), (zz, y1[yy], x1[xx]),
               (z1[zz], yy, xx), (z1[zz], yy, x1[xx]), (z1[zz], y1[yy], xx),
               (z1[zz], y1[yy], x1[xx])]
    ref = np.stack([a[c] for c in corners], axis=-1)
    np.testing.assert_array_equal(got, ref)
