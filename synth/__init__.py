"""Seeded synthetic workload generators (no SSA arithmetic). See generators.py."""
from .generators import (Workload, config1, config2, config3, config4, config5,  # noqa: F401
                         small_shaped, separable_image, draw_terms, disc_with_holes, get, CONFIGS)
