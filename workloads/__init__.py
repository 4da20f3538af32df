"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic)."""
from .ds import (C4_MATERIALS, DS_NCOMP, DS_RADIUS_MM, DS_SIZE_MM, DS_WEIGHT_PCT, GRAIN_DENSITY, M0,
                 Template, ds_number_fractions, ds_template, ds_templates, ds_type_counts,
                 sphere_template, union_mass_inertia)
from .scenes import (GID_STRIDE, INT64_MAX, MAT_A, MAT_B, Plane, Scene, box_planes, c1_box, c2_head_on,
                     c2_wall, c3_repose, load_scene, random_clumps, random_quaternions, random_spheres,
                     rsa_bed, save_scene, tile_scene)
