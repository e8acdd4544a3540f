// tsylv drop-in umbrella (B200 build): the reference's public header set
// (proj/include/tsylv/tsylv.hpp) for the Schur-basis solve path.
#pragma once
#include "tsylv/config.hpp"
#include "tsylv/errors.hpp"
#include "tsylv/gpu.hpp"
#include "tsylv/gsylv.hpp"
#include "tsylv/lapack.hpp"
#include "tsylv/laplace.hpp"
#include "tsylv/matrix.hpp"
#include "tsylv/oracle.hpp"
#include "tsylv/problems.hpp"
#include "tsylv/random.hpp"
#include "tsylv/scalar.hpp"
#include "tsylv/solvability.hpp"
#include "tsylv/sylvester.hpp"
#include "tsylv/tensor.hpp"
