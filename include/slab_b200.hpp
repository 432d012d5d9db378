/*
 * slab_b200.hpp — C++ facade over the C ABI (slab_b200.h) that mirrors the reference's operator
 * API (namespace slab, /root/reference/proj/include/slab/ *.hpp): same type and function names,
 * same argument order, same exceptions. A program written against slab:: switches to the GPU path
 * by including this header, `namespace slab = slab_b200;`, and creating one Context — see
 * INTEGRATION.md. Header-only; link with libslab_b200.so.
 *
 * Differences a port has to know about (all forced by the device boundary):
 *  - containers are opaque and GPU-resident: element access is explicit (values() downloads,
 *    DenseVector::from uploads); apply_masked (operations.hpp:136-143) takes an arbitrary host
 *    lambda and cannot cross a C ABI — its one use on the hot path, the Gauss-Seidel update, is
 *    fused into rbgs_color_step;
 *  - ProblemLevel owns a device hierarchy; `coarser()` is an accessor instead of a unique_ptr member;
 *  - LevelStats carries nnz_visited; the wall-clock fields are not filled inside CUDA graphs.
 */
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "slab_b200.h"

namespace slab_b200 {

	// ---- error.hpp:25-42
	struct Error : std::runtime_error {
		using std::runtime_error::runtime_error;
	};
	struct DimensionMismatch : Error {
		using Error::Error;
	};
	struct InvalidArgument : Error {
		using Error::Error;
	};
	struct SolverBreakdown : Error {
		using Error::Error;
	};
	struct CudaError : Error {
		using Error::Error;
	};

	namespace detail {
		inline void check( int status ) {
			if( status == SLAB_OK ) {
				return;
			}
			const std::string message = slab_last_error();
			switch( status ) {
				case SLAB_ERR_DIMENSION_MISMATCH: throw DimensionMismatch( message );
				case SLAB_ERR_INVALID_ARGUMENT: throw InvalidArgument( message );
				case SLAB_ERR_SOLVER_BREAKDOWN: throw SolverBreakdown( message );
				case SLAB_ERR_CUDA: throw CudaError( message );
				default: throw Error( message );
			}
		}
	} // namespace detail

	// ---- descriptor.hpp:26-38
	struct Descriptor {
		bool structural = false;
		bool transpose_matrix = false;
		unsigned flags() const noexcept {
			return ( structural ? SLAB_DESC_STRUCTURAL : 0u ) | ( transpose_matrix ? SLAB_DESC_TRANSPOSE : 0u );
		}
	};
	namespace descriptors {
		inline constexpr Descriptor none{};
		inline constexpr Descriptor structural{ true, false };
		inline constexpr Descriptor transpose_matrix{ false, true };
		inline constexpr Descriptor structural_transpose{ true, true };
	} // namespace descriptors

	/** One device + one stream; every container is created from a context. */
	class Context {
	public:
		explicit Context( int device = 0 ) {
			detail::check( slab_ctx_create( device, &ctx_ ) );
		}
		~Context() {
			slab_ctx_destroy( ctx_ );
		}
		Context( const Context & ) = delete;
		Context & operator=( const Context & ) = delete;
		slab_ctx_t handle() const noexcept {
			return ctx_;
		}
		void sync() const {
			detail::check( slab_ctx_sync( ctx_ ) );
		}
		/** SLAB_DOT_EXACT reproduces the reference's reduction order bit for bit; SLAB_DOT_TREE is faster. */
		void set_dot_mode( int mode ) {
			detail::check( slab_ctx_set_dot_mode( ctx_, mode ) );
		}

	private:
		slab_ctx_t ctx_ = nullptr;
	};

	// ---- dense_vector.hpp:33-66
	class DenseVector {
	public:
		DenseVector() = default;
		DenseVector( Context & ctx, std::size_t length, double value = 0.0 ) {
			detail::check( slab_vec_create( ctx.handle(), length, value, &v_ ) );
		}
		static DenseVector from( Context & ctx, const std::vector< double > & values ) {
			DenseVector v( ctx, values.size() );
			detail::check( slab_vec_upload( v.v_, values.data(), values.size() ) );
			return v;
		}
		~DenseVector() {
			if( owned_ ) {
				slab_vec_destroy( v_ );
			}
		}
		DenseVector( DenseVector && other ) noexcept : v_( other.v_ ), owned_( other.owned_ ) {
			other.v_ = nullptr;
		}
		DenseVector & operator=( DenseVector && other ) noexcept {
			if( this != &other ) {
				if( owned_ ) {
					slab_vec_destroy( v_ );
				}
				v_ = other.v_;
				owned_ = other.owned_;
				other.v_ = nullptr;
			}
			return *this;
		}
		DenseVector( const DenseVector & ) = delete;
		DenseVector & operator=( const DenseVector & ) = delete;

		std::size_t size() const {
			uint64_t n = 0;
			if( v_ ) {
				detail::check( slab_vec_size( v_, &n ) );
			}
			return n;
		}
		/** Downloads the values in the reference's natural ordering. */
		std::vector< double > values() const {
			std::vector< double > out( size() );
			detail::check( slab_vec_download( v_, out.data(), out.size() ) );
			return out;
		}
		void assign( const std::vector< double > & values ) {
			detail::check( slab_vec_upload( v_, values.data(), values.size() ) );
		}
		bool operator==( const DenseVector & other ) const {
			return values() == other.values();
		}
		slab_vec_t handle() const noexcept {
			return v_;
		}
		static DenseVector borrow( slab_vec_t handle ) {
			DenseVector v;
			v.v_ = handle;
			v.owned_ = false;
			return v;
		}

	private:
		slab_vec_t v_ = nullptr;
		bool owned_ = true;
	};

	// ---- sparse_matrix.hpp:31-171
	struct Triplet {
		std::size_t row = 0;
		std::size_t col = 0;
		double value = 0.0;
	};

	class SparseMatrix {
	public:
		SparseMatrix() = default;
		static SparseMatrix from_csr( Context & ctx, std::size_t nrows, std::size_t ncols,
			const std::vector< std::size_t > & row_offsets, const std::vector< std::size_t > & col_indices,
			const std::vector< double > & values ) {
			if( row_offsets.size() != nrows + 1 || row_offsets.front() != 0 ) {
				throw InvalidArgument( "from_csr: row_offsets must have nrows+1 entries starting at 0" );
			}
			if( row_offsets.back() != col_indices.size() || col_indices.size() != values.size() ) {
				throw InvalidArgument( "from_csr: offsets, column and value arrays disagree on nnz" );
			}
			const std::vector< uint64_t > ro( row_offsets.begin(), row_offsets.end() ), co( col_indices.begin(), col_indices.end() );
			SparseMatrix A;
			detail::check( slab_mat_create_csr( ctx.handle(), nrows, ncols, ro.data(), co.data(), values.data(), &A.m_ ) );
			return A;
		}
		~SparseMatrix() {
			if( owned_ ) {
				slab_mat_destroy( m_ );
			}
		}
		SparseMatrix( SparseMatrix && other ) noexcept : m_( other.m_ ), owned_( other.owned_ ) {
			other.m_ = nullptr;
		}
		SparseMatrix & operator=( SparseMatrix && other ) noexcept {
			if( this != &other ) {
				if( owned_ ) {
					slab_mat_destroy( m_ );
				}
				m_ = other.m_;
				owned_ = other.owned_;
				other.m_ = nullptr;
			}
			return *this;
		}
		SparseMatrix( const SparseMatrix & ) = delete;
		SparseMatrix & operator=( const SparseMatrix & ) = delete;

		std::size_t nrows() const {
			uint64_t v = 0;
			detail::check( slab_mat_shape( m_, &v, nullptr, nullptr ) );
			return v;
		}
		std::size_t ncols() const {
			uint64_t v = 0;
			detail::check( slab_mat_shape( m_, nullptr, &v, nullptr ) );
			return v;
		}
		std::size_t nnz() const {
			uint64_t v = 0;
			detail::check( slab_mat_shape( m_, nullptr, nullptr, &v ) );
			return v;
		}
		// how the matrix is held on the device: plain SELL-32 only, or with the dictionary-coded copy
		slab_format_info format_info() const {
			slab_format_info info{};
			detail::check( slab_mat_format_info( m_, &info ) );
			return info;
		}
		slab_mat_t handle() const noexcept {
			return m_;
		}
		static SparseMatrix adopt( slab_mat_t handle, bool owned ) {
			SparseMatrix A;
			A.m_ = handle;
			A.owned_ = owned;
			return A;
		}

	private:
		slab_mat_t m_ = nullptr;
		bool owned_ = true;
	};

	// ---- index_mask.hpp:35-73
	class IndexMask {
	public:
		IndexMask( Context & ctx, std::size_t universe_size, std::vector< std::size_t > members )
			: universe_( universe_size ), members_( std::move( members ) ) {
			const std::vector< uint64_t > m( members_.begin(), members_.end() );
			detail::check( slab_mask_create( ctx.handle(), universe_size, m.data(), m.size(), &h_ ) );
		}
		~IndexMask() {
			slab_mask_destroy( h_ );
		}
		IndexMask( const IndexMask & ) = delete;
		IndexMask & operator=( const IndexMask & ) = delete;
		std::size_t universe_size() const noexcept {
			return universe_;
		}
		const std::vector< std::size_t > & members() const noexcept {
			return members_;
		}
		std::size_t size() const noexcept {
			return members_.size();
		}
		slab_mask_t handle() const noexcept {
			return h_;
		}

	private:
		slab_mask_t h_ = nullptr;
		std::size_t universe_ = 0;
		std::vector< std::size_t > members_;
	};

	// ---- operations.hpp:49-230
	inline DenseVector & set_all( DenseVector & v, double value ) {
		detail::check( slab_set_all( v.handle(), value ) );
		return v;
	}
	inline double dot( const DenseVector & x, const DenseVector & y ) {
		double out = 0.0;
		detail::check( slab_dot( x.handle(), y.handle(), &out ) );
		return out;
	}
	inline DenseVector & waxpby( DenseVector & w, double alpha, const DenseVector & x, double beta, const DenseVector & y ) {
		detail::check( slab_waxpby( w.handle(), alpha, x.handle(), beta, y.handle() ) );
		return w;
	}
	inline DenseVector & mxv( DenseVector & y, const SparseMatrix & A, const DenseVector & x, Descriptor desc = {} ) {
		detail::check( slab_mxv( y.handle(), A.handle(), x.handle(), desc.flags() ) );
		return y;
	}
	inline DenseVector & mxv( DenseVector & y, const IndexMask & mask, const SparseMatrix & A, const DenseVector & x,
		Descriptor desc = {} ) {
		detail::check( slab_mxv_masked( y.handle(), mask.handle(), A.handle(), x.handle(), desc.flags() ) );
		return y;
	}

	// ---- problem.hpp
	struct GridDims {
		std::size_t nx = 0, ny = 0, nz = 0;
		std::size_t n() const noexcept {
			return nx * ny * nz;
		}
		bool operator==( const GridDims & ) const = default;
	};
	struct LevelStats { // problem.hpp:204-209
		std::uint64_t smoother_ns = 0, transfer_ns = 0, mg_ns = 0, nnz_visited = 0;
	};

	inline SparseMatrix build_matrix( Context & ctx, const GridDims & dims ) { // problem.hpp:90-131
		slab_mat_t m = nullptr;
		detail::check( slab_mat_create_stencil27( ctx.handle(), dims.nx, dims.ny, dims.nz, &m ) );
		return SparseMatrix::adopt( m, true );
	}
	inline SparseMatrix build_restriction( Context & ctx, const GridDims & fine ) { // problem.hpp:174-201
		slab_mat_t m = nullptr;
		detail::check( slab_mat_create_restriction( ctx.handle(), fine.nx, fine.ny, fine.nz, &m ) );
		return SparseMatrix::adopt( m, true );
	}
	inline DenseVector build_rhs( Context & ctx, const GridDims & dims ) { // problem.hpp:134-137
		if( dims.nx < 2 || dims.ny < 2 || dims.nz < 2 ) {
			throw InvalidArgument( "grid dimensions must all be at least 2" );
		}
		return DenseVector( ctx, dims.n(), 1.0 );
	}

	/** problem.hpp:220-277. Owns the device hierarchy when created by build_hierarchy / from a matrix. */
	class ProblemLevel {
	public:
		ProblemLevel() = default;
		/** Standalone level around an arbitrary square CSR system (problem.hpp:253). */
		ProblemLevel( Context & ctx, std::size_t n, const std::vector< std::size_t > & row_offsets,
			const std::vector< std::size_t > & col_indices, const std::vector< double > & values ) {
			const std::vector< uint64_t > ro( row_offsets.begin(), row_offsets.end() ), co( col_indices.begin(), col_indices.end() );
			detail::check( slab_level_create_csr( ctx.handle(), n, ro.data(), co.data(), values.data(), &h_ ) );
		}
		~ProblemLevel() {
			if( owned_ ) {
				slab_level_destroy( h_ );
			}
		}
		ProblemLevel( ProblemLevel && other ) noexcept : h_( other.h_ ), owned_( other.owned_ ) {
			other.h_ = nullptr;
		}
		ProblemLevel & operator=( ProblemLevel && other ) noexcept {
			if( this != &other ) {
				if( owned_ ) {
					slab_level_destroy( h_ );
				}
				h_ = other.h_;
				owned_ = other.owned_;
				other.h_ = nullptr;
			}
			return *this;
		}
		ProblemLevel( const ProblemLevel & ) = delete;
		ProblemLevel & operator=( const ProblemLevel & ) = delete;

		std::size_t n() const {
			uint64_t v = 0;
			detail::check( slab_level_info( h_, nullptr, &v, nullptr, nullptr, nullptr ) );
			return v;
		}
		GridDims dims() const {
			uint64_t d[ 3 ] = { 0, 0, 0 };
			detail::check( slab_level_info( h_, d, nullptr, nullptr, nullptr, nullptr ) );
			return { d[ 0 ], d[ 1 ], d[ 2 ] };
		}
		std::size_t depth() const {
			uint64_t v = 0;
			detail::check( slab_level_info( h_, nullptr, nullptr, nullptr, nullptr, &v ) );
			return v;
		}
		std::size_t num_colors() const {
			uint64_t v = 0;
			detail::check( slab_level_info( h_, nullptr, nullptr, nullptr, &v, nullptr ) );
			return v;
		}
		bool has_coarser() const {
			slab_level_t c = nullptr;
			detail::check( slab_level_coarser( h_, &c ) );
			return c != nullptr;
		}
		ProblemLevel coarser() const { // borrowed view of *level.coarser
			ProblemLevel out;
			detail::check( slab_level_coarser( h_, &out.h_ ) );
			out.owned_ = false;
			return out;
		}
		SparseMatrix A() const {
			slab_mat_t m = nullptr;
			detail::check( slab_level_matrix( h_, &m ) );
			return SparseMatrix::adopt( m, false );
		}
		std::optional< SparseMatrix > restriction() const {
			slab_mat_t m = nullptr;
			detail::check( slab_level_restriction( h_, &m ) );
			if( m == nullptr ) {
				return std::nullopt;
			}
			return SparseMatrix::adopt( m, false );
		}
		DenseVector a_diag() const {
			slab_vec_t v = nullptr;
			detail::check( slab_level_diag( h_, &v ) );
			return DenseVector::borrow( v );
		}
		std::vector< std::size_t > color_members( std::size_t k ) const { // colors.masks[k].members()
			uint64_t size = 0;
			detail::check( slab_level_color_info( h_, k, &size, nullptr ) );
			std::vector< uint64_t > m( size );
			detail::check( slab_level_color_members( h_, k, m.data() ) );
			return { m.begin(), m.end() };
		}
		std::uint64_t color_nnz( std::size_t k ) const {
			uint64_t v = 0;
			detail::check( slab_level_color_info( h_, k, nullptr, &v ) );
			return v;
		}
		// how the colour-major matrix copy the smoother reads is held on the device (slab_b200.h: slab_format_info)
		slab_format_info format_info() const {
			slab_format_info info{};
			detail::check( slab_level_format_info( h_, &info ) );
			return info;
		}
		LevelStats stats() const {
			slab_level_stats s{};
			detail::check( slab_level_stats_get( h_, &s ) );
			return { s.smoother_ns, s.transfer_ns, s.mg_ns, s.nnz_visited };
		}
		void reset_stats() {
			detail::check( slab_level_stats_reset( h_ ) );
		}
		slab_level_t handle() const noexcept {
			return h_;
		}
		static ProblemLevel adopt( slab_level_t h ) {
			ProblemLevel L;
			L.h_ = h;
			return L;
		}

	private:
		slab_level_t h_ = nullptr;
		bool owned_ = true;
	};

	inline ProblemLevel build_hierarchy( Context & ctx, const GridDims & dims, std::size_t levels ) { // problem.hpp:284-319
		slab_level_t h = nullptr;
		detail::check( slab_hierarchy_create( ctx.handle(), dims.nx, dims.ny, dims.nz, levels, &h ) );
		return ProblemLevel::adopt( h );
	}

	// ---- smoother.hpp
	struct SmootherConfig {
		std::size_t sweeps = 1;
	};
	inline DenseVector & rbgs_forward( ProblemLevel & level, DenseVector & z, const DenseVector & r ) {
		detail::check( slab_rbgs_forward( level.handle(), z.handle(), r.handle() ) );
		return z;
	}
	inline DenseVector & rbgs_backward( ProblemLevel & level, DenseVector & z, const DenseVector & r ) {
		detail::check( slab_rbgs_backward( level.handle(), z.handle(), r.handle() ) );
		return z;
	}
	inline DenseVector & rbgs_symmetric( ProblemLevel & level, DenseVector & z, const DenseVector & r,
		const SmootherConfig & cfg = {} ) {
		if( cfg.sweeps < 1 ) {
			throw InvalidArgument( "SmootherConfig: sweeps must be at least 1" );
		}
		detail::check( slab_rbgs_symmetric( level.handle(), z.handle(), r.handle(), cfg.sweeps ) );
		return z;
	}
	namespace detail {
		inline void rbgs_color_step( ProblemLevel & level, std::size_t k, DenseVector & z, const DenseVector & r ) {
			check( slab_rbgs_color_step( level.handle(), k, z.handle(), r.handle() ) );
		}
		// extension: the step twice in a row as one launch (the turnaround of rbgs_symmetric)
		inline void rbgs_color_step_twice( ProblemLevel & level, std::size_t k, DenseVector & z, const DenseVector & r ) {
			check( slab_rbgs_color_step_twice( level.handle(), k, z.handle(), r.handle() ) );
		}
	} // namespace detail

	// ---- multigrid.hpp
	inline void restrict_vector( ProblemLevel & level, const DenseVector & v_fine, DenseVector & out ) {
		detail::check( slab_restrict_vector( level.handle(), v_fine.handle(), out.handle() ) );
	}
	inline DenseVector & refine_and_add( ProblemLevel & level, DenseVector & z, const DenseVector & z_c ) {
		detail::check( slab_refine_and_add( level.handle(), z.handle(), z_c.handle() ) );
		return z;
	}
	inline DenseVector & mg_vcycle( ProblemLevel & level, DenseVector & z, const DenseVector & r,
		const SmootherConfig & smoother_cfg = {} ) {
		if( smoother_cfg.sweeps < 1 ) {
			throw InvalidArgument( "SmootherConfig: sweeps must be at least 1" );
		}
		detail::check( slab_mg_vcycle( level.handle(), z.handle(), r.handle(), smoother_cfg.sweeps ) );
		return z;
	}

	// ---- cg.hpp
	struct CGConfig {
		std::size_t max_iters = 500;
		double rtol = 1e-6;
		bool use_preconditioner = true;
		std::optional< std::size_t > fixed_iterations;
	};
	struct CGResult {
		std::size_t iterations = 0;
		std::vector< double > residual_history;
		bool converged = false;
		DenseVector solution;
		double solve_ms = 0.0; ///< device time of the solve (CUDA events); not in the reference
	};
	inline double residual_norm( const SparseMatrix & A, const DenseVector & x, const DenseVector & b ) {
		double out = 0.0;
		detail::check( slab_residual_norm( A.handle(), x.handle(), b.handle(), &out ) );
		return out;
	}
	inline CGResult cg_solve( Context & ctx, ProblemLevel & hierarchy, const DenseVector & b, const DenseVector & x0,
		const CGConfig & cfg = {}, const SmootherConfig & smoother_cfg = {} ) {
		slab_cg_config c;
		slab_cg_config_default( &c );
		c.max_iters = cfg.max_iters;
		c.rtol = cfg.rtol;
		c.use_preconditioner = cfg.use_preconditioner ? 1 : 0;
		c.has_fixed_iterations = cfg.fixed_iterations ? 1 : 0;
		c.fixed_iterations = cfg.fixed_iterations.value_or( 0 );
		c.sweeps = smoother_cfg.sweeps;
		CGResult out;
		out.solution = DenseVector( ctx, hierarchy.n() );
		std::vector< double > history( ( cfg.max_iters > 0 ? cfg.max_iters : 1 ) + 1, 0.0 );
		slab_cg_result res{};
		detail::check( slab_cg_solve( hierarchy.handle(), b.handle(), x0.handle(), &c, out.solution.handle(), history.data(),
			&res ) );
		out.iterations = res.iterations;
		out.converged = res.converged != 0;
		out.solve_ms = res.solve_ms;
		history.resize( res.iterations + 1 );
		out.residual_history = std::move( history );
		return out;
	}

	// ---- bench.hpp:53-105 — the HPCG symmetry test (caller of the hot path)
	struct SymmetryReport { // report.hpp:63-75
		bool skipped = false;
		bool matrix_pass = false;
		double matrix_diff = 0.0;
		bool precond_pass = false;
		double precond_diff = 0.0;
		double tolerance = 0.0;
		bool all_pass() const noexcept {
			return skipped || ( matrix_pass && precond_pass );
		}
	};
	inline double symmetry_tolerance( const DenseVector & x, const DenseVector & y ) { // bench.hpp:53-57
		const double nx = std::sqrt( dot( x, x ) );
		const double ny = std::sqrt( dot( y, y ) );
		return 1e-8 * nx * ny * 26.0 * std::sqrt( static_cast< double >( x.size() ) );
	}
	namespace detail {
		template< class Apply >
		inline double bilinear_asymmetry( Context & ctx, Apply && apply, const DenseVector & x, const DenseVector & y ) {
			DenseVector tmp( ctx, x.size() ); // bench.hpp:63-70
			apply( tmp, y );
			const double lhs = dot( x, tmp );
			apply( tmp, x );
			const double rhs = dot( y, tmp );
			return std::abs( lhs - rhs );
		}
	} // namespace detail

	// ---- rng.hpp:35-65 (host generator, then upload)
	class Lcg64 {
	public:
		explicit Lcg64( std::uint64_t seed ) : state_( seed ) {}
		std::uint64_t next_u64() {
			state_ = state_ * 6364136223846793005ULL + 1442695040888963407ULL;
			return state_;
		}
		double next_unit() {
			return static_cast< double >( next_u64() >> 11 ) * 0x1.0p-53;
		}
		double next_symmetric() {
			return 2.0 * next_unit() - 1.0;
		}

	private:
		std::uint64_t state_;
	};
	inline DenseVector random_vector( Context & ctx, std::size_t n, Lcg64 & rng ) {
		std::vector< double > host( n );
		for( std::size_t i = 0; i < n; ++i ) {
			host[ i ] = rng.next_symmetric();
		}
		return DenseVector::from( ctx, host );
	}

	/** bench.hpp:80-105: operator and V-cycle must act symmetrically on two LCG vectors. */
	inline SymmetryReport symmetry_test( Context & ctx, ProblemLevel & hierarchy, std::uint64_t seed,
		const SmootherConfig & smoother_cfg = {} ) {
		const std::size_t n = hierarchy.n();
		Lcg64 rng( seed );
		const DenseVector x = random_vector( ctx, n, rng );
		const DenseVector y = random_vector( ctx, n, rng );
		SymmetryReport out;
		out.tolerance = symmetry_tolerance( x, y );
		const SparseMatrix A = hierarchy.A();
		out.matrix_diff = detail::bilinear_asymmetry(
			ctx, [ &A ]( DenseVector & result, const DenseVector & in ) { mxv( result, A, in ); }, x, y );
		out.matrix_pass = out.matrix_diff <= out.tolerance;
		out.precond_diff = detail::bilinear_asymmetry(
			ctx,
			[ &hierarchy, &smoother_cfg ]( DenseVector & result, const DenseVector & in ) {
				set_all( result, 0.0 );
				mg_vcycle( hierarchy, result, in, smoother_cfg );
			},
			x, y );
		out.precond_pass = out.precond_diff <= out.tolerance;
		return out;
	}

} // namespace slab_b200
