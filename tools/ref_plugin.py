"""pytest plugin: run the reference's OWN tests with its batch-level entry
points routed to this package ("Implication for the
build"): vdikit.generate_vdi and vdikit.render_vdi (and every module that
imported them by name) become paper_2206_08660_b200.generate_vdi /
render_vdi before the test modules import them. The reference's single-ray
helpers (generate_list, find_gamma, dda_traverse, ...) and its DVR, preview,
codec and metrics stay the reference's CPU code, so the tests compare the
B200 batch path against the reference's own ground truths.

    PYTHONPATH=<vdikit src>:<repo> python -m pytest -p tools.ref_plugin <vdikit tests> ...

At the end the plugin prints how many calls went to the B200 path (a run
where they stayed zero did not test it).
"""

import vdikit
import vdikit.client
import vdikit.generate
import vdikit.raycast

import paper_2206_08660_b200 as vb

CALLS = {"generate_vdi": 0, "render_vdi": 0}


def generate_vdi(vol, tf, cam, params=None, grid_dims=None, with_stats=False):
    CALLS["generate_vdi"] += 1
    return vb.generate_vdi(vol, tf, cam, params, grid_dims, with_stats)


def render_vdi(vdi, grid, cam_new, opts=None, with_stats=False):
    CALLS["render_vdi"] += 1
    return vb.render_vdi(vdi, grid, cam_new, opts, with_stats)


for mod in (vdikit, vdikit.generate):
    mod.generate_vdi = generate_vdi
for mod in (vdikit, vdikit.raycast, vdikit.client):
    mod.render_vdi = render_vdi


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(
        f"B200 drop-in calls: generate_vdi {CALLS['generate_vdi']}, "
        f"render_vdi {CALLS['render_vdi']}")
