"""B200-native CVO registration engine (drop-in for the kreg hot path)."""
from .types import *  # noqa: F401,F403
