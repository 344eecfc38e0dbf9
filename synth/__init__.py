"""Seeded synthetic input generators (no method arithmetic); see synth/generators.py."""
from .generators import *  # noqa: F401,F403
