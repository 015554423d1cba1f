from .sequence import *  # noqa
