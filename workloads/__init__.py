"""Seeded input generators (no sorting arithmetic). See gen.py."""
