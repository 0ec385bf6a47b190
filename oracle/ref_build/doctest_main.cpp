#include <doctest.h>
